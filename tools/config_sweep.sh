#!/bin/bash
# Bench lines for the other BASELINE configs / options (no e2e, no cpu baseline)
out=${SWEEP_OUT:-gpurun_out/sweep}
mkdir -p $out
for spec in "c1 f64 0" "c2 f64 0" "c2 f32 0" "c3 f64 0" "c3hi f64 0" "c5 f64 0" "c6 f64 0" "r22 f64 0" "c4 f32 0" "c4 f64 1"; do
  set -- $spec
  python bench.py --config $1 --dtype $2 --refresh $3 --no-e2e --no-cpu --no-random-ids --no-ari --passes 3 --steps 30 --warmup 3 \
    > $out/$1_$2_r$3.json 2> $out/$1_$2_r$3.err
  echo "$1 $2 refresh=$3 rc=$?"
done

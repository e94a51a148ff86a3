#!/bin/bash
# A/B of an env switch on graph-launched iteration time (one process per setting).
# usage: VAR=OFSC_C3_CTAS AB_SET="2 3" tools/conc_ab.sh c4 c5   (any env switch of the library)
var=${VAR:?set VAR to the env switch to A/B}
out=${AB_OUT:-gpurun_out/ab.jsonl}
for v in ${AB_SET:-0 1 0 1}; do
  env $var=$v ITER_TAG="$var=$v" python tools/iter_time.py "$@" >> $out 2>>${out%.jsonl}.err
done
cat $out

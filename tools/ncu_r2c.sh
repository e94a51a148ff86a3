#!/bin/bash
# Round-2 closing pass: full GPU suite, bench, bench launch list under ncu, and one
# ncu --set full capture of a late K-means light step.  Outputs in gpurun_out/r2c.
out=gpurun_out/r2c
mkdir -p $out
timeout 600 python __graft_entry__.py smoke > $out/smoke.log 2>&1; echo smoke=$? >> $out/status.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $out/tests.log 2>&1; echo tests=$? >> $out/status.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo bench=$? >> $out/status.txt
B="bench.py --steps 2 --warmup 3 --no-cpu --no-methods --no-random-ids --passes 1 --e2e-steps 1"
python $B > $out/plain_bench.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches.csv python $B > $out/launches_bench.log 2>&1
echo launches=$? >> $out/status.txt
python tools/kmeans_feat_probe.py c4 > $out/plain_km.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_kmeans_light -s 60 -c 1 \
    -o $out/km_light_full python tools/kmeans_feat_probe.py c4 > $out/km_light_full.log 2>&1
echo full_km_light=$? >> $out/status.txt

#!/bin/bash
# A/B of an env switch on graph-launched iteration time (one process per setting).
# usage: VAR=OFSC_EXP_CONC tools/conc_ab.sh c4 c5
var=${VAR:-OFSC_EXP_CONC}
out=${AB_OUT:-gpurun_out/ab.jsonl}
for v in ${AB_SET:-0 1 0 1}; do
  env $var=$v ITER_TAG="$var=$v" python tools/iter_time.py "$@" >> $out 2>>${out%.jsonl}.err
done
cat $out

#!/bin/bash
# Per-iteration graph time with and without programmatic dependent launch (OFSC_PDL),
# one process per setting (the switch is read once per process).
out=${PDL_OUT:-gpurun_out/pdl}
mkdir -p $out
for pdl in ${PDL_SET:-0 1 0 1}; do
  OFSC_PDL=$pdl python tools/phase_time.py c1 c2 c3 c5 > $out/pdl$pdl.jsonl.tmp 2>&1
  cat $out/pdl$pdl.jsonl.tmp | sed "s/^{/{\"pdl\": $pdl, /" >> $out/pdl_ab.jsonl
done
rm -f $out/*.tmp

#!/bin/bash
out=gpurun_out/l2probe
mkdir -p $out
for v in ${VARIANTS:-base intra eq intra_eq small_blocks}; do
  VARIANT=$v timeout 300 python tools/l2_probe.py > $out/$v.txt 2>&1
  VARIANT=$v timeout 400 ncu --kernel-name regex:k_spmm --clock-control none --launch-skip 1 -c 1 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --csv python tools/l2_probe.py > $out/$v.csv 2>&1
  echo "$v rc=$?"
done

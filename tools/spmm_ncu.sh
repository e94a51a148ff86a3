#!/bin/bash
# DRAM bytes / duration / L2 hit rate of the SpMM (C2a) launches at c4 per column window.
out=gpurun_out/spmm_ncu
mkdir -p $out
for cw in ${CWS:-64 32 16}; do
  OFSC_SPMM_CW=$cw timeout 900 ncu --kernel-name regex:k_spmm --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -c ${NCU_COUNT:-8} --csv python tools/run_iters.py c4 3 > $out/cw$cw.csv 2> $out/cw$cw.err
  echo "cw=$cw rc=$?"
done

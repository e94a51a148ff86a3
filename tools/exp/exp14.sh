for rep in 1 2; do for cs in 0 1; do
  OFSC_SPMM_CS=$cs python tools/spmm_time.py c4 c5 c6 2>/dev/null | sed "s/^{/{\"cs\": $cs, /" >> gpurun_out/spmm_cs_ab.jsonl
done; done
for cs in 0 1 0 1; do OFSC_SPMM_CS=$cs ITER_METHODS=ofm_f2 ITER_TAG="cs=$cs" python tools/iter_time.py c4 >> gpurun_out/spmm_cs_iter.jsonl 2>/dev/null; done
for cs in 0 1; do OFSC_SPMM_CS=$cs timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_spmm -s 4 -c 2 --csv python tools/run_iters.py c4 3 > gpurun_out/spmm_cs_ncu_$cs.csv 2>/dev/null; done

#!/bin/bash
# Round-2 final profile pass (B200_PROFILING.md): each command plain first (exit 0),
# then under ncu.  Outputs in gpurun_out/r2prof_b.
out=gpurun_out/r2prof_b
mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
for m in ofm_f2 ofm_f1; do
  python tools/run_iters.py c4 3 $m > $out/plain_iters_$m.log 2>&1 && \
    timeout 900 ncu --clock-control none --metrics $M --csv python tools/run_iters.py c4 3 $m > $out/iter_metrics_$m.csv 2> $out/iter_metrics_$m.err
  echo metrics_$m=$? >> $out/status.txt
done
B="bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-methods --no-random-ids --no-ari --passes 1"
python $B > $out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches.csv python $B > $out/launches_bench.log 2>&1
echo launches=$? >> $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 \
  -o $out/spmm_full python tools/run_iters.py c4 3 > $out/spmm_full.log 2>&1
echo full_spmm=$? >> $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direction -s 2 -c 1 \
  -o $out/c3_full python tools/run_iters.py c4 3 > $out/c3_full.log 2>&1
echo full_c3=$? >> $out/status.txt
python tools/kmeans_feat_probe.py c4 > $out/plain_km.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:k_kmeans_step -s 60 -c 1 \
    -o $out/km_full python tools/kmeans_feat_probe.py c4 > $out/km_full.log 2>&1
echo full_km=$? >> $out/status.txt

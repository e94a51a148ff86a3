#!/bin/bash
# Per-kernel ncu metrics of one OFM-f2 iteration at c4 (launches of the 2nd iteration),
# then the launch list of bench.py (gpu__time_duration, B200_PROFILING.md pass).
out=gpurun_out/ncu_iter
mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --clock-control none --metrics $M --csv python tools/run_iters.py c4 3 > $out/iter_metrics.csv 2> $out/iter_metrics.err
echo metrics=$?
if [ "${LAUNCHES:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-methods > $out/launches_bench.log 2>&1
  echo launches=$?
fi

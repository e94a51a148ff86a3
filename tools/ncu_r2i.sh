#!/bin/bash
# Round-2 closing pass after the f1 diagonal C2b: smoke, full GPU suite, bench, bench
# launch list under ncu, per-kernel ncu metrics of one OFM-f1 and one OFM-f2 iteration
# at c4, and one ncu --set full capture of k_gram_diag.  Outputs in gpurun_out/r2i.
out=gpurun_out/r2i
mkdir -p $out
timeout 600 python __graft_entry__.py smoke > $out/smoke.log 2>&1; echo smoke=$? >> $out/status.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $out/tests.log 2>&1; echo tests=$? >> $out/status.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo bench=$? >> $out/status.txt
B="bench.py --steps 2 --warmup 3 --no-cpu --no-methods --no-random-ids --passes 1 --e2e-steps 1"
python $B > $out/plain_bench.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches.csv python $B > $out/launches_bench.log 2>&1
echo launches=$? >> $out/status.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
for m in ofm_f1 ofm_f2; do
  python tools/run_iters.py c4 3 $m > $out/plain_iter_$m.log 2>&1 && \
    timeout 900 ncu --clock-control none --metrics $M --csv python tools/run_iters.py c4 3 $m > $out/iter_metrics_$m.csv 2> $out/iter_metrics_$m.err
  echo iter_$m=$? >> $out/status.txt
done
python tools/run_iters.py c4 3 ofm_f1 > $out/plain_diag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_diag -s 1 -c 1 \
    -o $out/gram_diag_full python tools/run_iters.py c4 3 ofm_f1 > $out/gram_diag_full.log 2>&1
echo full_gram_diag=$? >> $out/status.txt
cat $out/status.txt

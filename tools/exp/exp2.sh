set -x
timeout 900 python -m pytest tests/test_gpu_cluster.py -q -x -p no:cacheprovider -k "kmeans" > gpurun_out/exp2_tests.log 2>&1; tail -5 gpurun_out/exp2_tests.log
OFSC_KMEANS_STATS=1 E2E_REPS=1 timeout 300 python tools/e2e_trace.py c4 > gpurun_out/km_stats2.log 2>&1
E2E_REPS=3 OFSC_TRACE=2 timeout 300 python tools/e2e_trace.py c4 > gpurun_out/e2e_trace2.log 2>&1

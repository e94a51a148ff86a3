set -x
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/exp3_tests.log 2>&1; tail -3 gpurun_out/exp3_tests.log
OFSC_KMEANS_STATS=1 E2E_REPS=2 timeout 300 python tools/e2e_trace.py c4 > gpurun_out/km_stats3.log 2>&1
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err

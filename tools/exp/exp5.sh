set -x
timeout 1500 python -m pytest tests/test_gpu_iterate.py tests/test_gpu_production.py tests/test_gpu_stream.py -q -x -p no:cacheprovider > gpurun_out/exp5_tests.log 2>&1; tail -3 gpurun_out/exp5_tests.log

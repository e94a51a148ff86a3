set -x
timeout 600 python __graft_entry__.py smoke > gpurun_out/exp8_smoke.log 2>&1; tail -2 gpurun_out/exp8_smoke.log
timeout 1500 python -m pytest tests/test_gpu_iterate.py -q -x -p no:cacheprovider > gpurun_out/exp8_tests.log 2>&1; tail -3 gpurun_out/exp8_tests.log
for v in 1 0 1 0; do OFSC_SMALL=$v ITER_METHODS=ofm_f1,triofm_f1,ofm_f2,triofm_f2 ITER_TAG="small=$v" timeout 600 python tools/iter_time.py c1 c2 >> gpurun_out/small_ab.jsonl 2>>gpurun_out/small_ab.err; done

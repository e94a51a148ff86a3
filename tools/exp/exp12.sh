timeout 900 python -m pytest tests/test_gpu_iterate.py -q -x -p no:cacheprovider -k "c3_kernel_variants or p2_ten" > gpurun_out/exp12_tests.log 2>&1; tail -2 gpurun_out/exp12_tests.log
for rep in 1 2; do for ws in 0 2; do
  OFSC_C3_WS=$ws ITER_METHODS=ofm_f2,triofm_f2 ITER_TAG="ws=$ws" timeout 600 python tools/iter_time.py c4 c5 c3 >> gpurun_out/c3wg_ab.jsonl 2>>gpurun_out/c3wg_ab.err
done; done
for ws in 0 2; do OFSC_C3_WS=$ws ITER_METHODS=ofm_f2,triofm_f2 timeout 600 python tools/method_ab.py c4 > gpurun_out/c3wg_method_$ws.jsonl 2>&1; done

set -x
timeout 900 python -m pytest tests/test_gpu_iterate.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "c3_kernel_variants or kmeans" > gpurun_out/exp7_tests.log 2>&1; tail -3 gpurun_out/exp7_tests.log
for rep in 1 2; do
for c in x 3; do
  if [ "$c" = "x" ]; then unset OFSC_C3_CTAS; else export OFSC_C3_CTAS=$c; fi
  ITER_METHODS=ofm_f1,triofm_f1,ofm_f2,triofm_f2 ITER_TAG="ctas=$c" timeout 600 python tools/iter_time.py c5 c2 >> gpurun_out/c3_grid_f1_ab.jsonl 2>>gpurun_out/c3_grid_f1_ab.err
done
done

set -x
timeout 900 python -m pytest tests/test_gpu_iterate.py -q -x -p no:cacheprovider -k "c3_kernel_variants" > gpurun_out/exp6_tests.log 2>&1; tail -3 gpurun_out/exp6_tests.log
for rep in 1 2; do
for cfg in "0 x" "1 x" "0 2" "1 2" "0 3" "1 3"; do
  set -- $cfg
  if [ "$2" = "x" ]; then unset OFSC_C3_CTAS; else export OFSC_C3_CTAS=$2; fi
  OFSC_C3_SPLIT=$1 ITER_METHODS=ofm_f2,triofm_f2 ITER_TAG="split=$1 ctas=$2" timeout 600 python tools/iter_time.py c5 c4 >> gpurun_out/c3split2_ab.jsonl 2>>gpurun_out/c3split2_ab.err
done
done

set -x
timeout 900 python -m pytest tests/test_gpu_iterate.py -q -x -p no:cacheprovider -k "c3_kernel_variants or p2 or P2 or one_step" > gpurun_out/exp4_tests.log 2>&1; tail -3 gpurun_out/exp4_tests.log
ITER_METHODS=ofm_f2,triofm_f2 AB_OUT=gpurun_out/c3split_ab.jsonl AB_SET="0 1 0 1" VAR=OFSC_C3_SPLIT timeout 1200 tools/conc_ab.sh c4 c5 c3
for v in 0 1; do OFSC_C3_SPLIT=$v timeout 600 python tools/method_ab.py c4 > gpurun_out/c3split_method_$v.jsonl 2>&1; done

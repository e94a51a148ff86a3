#!/bin/bash
# compute-sanitizer on small cases (SURVEY sec. 4 layer 7), ONE tool per gpurun call:
#   bash tools/sanitize.sh memcheck|racecheck|synccheck
# The same pytest selection runs plain first (exit 0) before the sanitizer.
tool=${1:-memcheck}
out=gpurun_out/r2san
mkdir -p $out
SEL="tests/test_gpu_iterate.py::test_p1_one_step
 tests/test_gpu_iterate.py::test_p2_wide_kernels[ofm_f2-64]
 tests/test_gpu_iterate.py::test_p2_wide_kernels[triofm_f1-48]
 tests/test_gpu_kernels.py::test_fused_spmm_gram
 tests/test_gpu_kernels.py::test_spmm_production_variants
 tests/test_gpu_cluster.py::test_kmeans_fused_step_shapes
 tests/test_gpu_cluster.py::test_algorithm1_end_to_end_c1
 tests/test_gpu_multirank.py::test_p5_ten_steps_vs_oracle[ofm_f2-2]"
python -m pytest $SEL -q -x -p no:cacheprovider > $out/plain_$tool.log 2>&1 || { echo "plain run failed" > $out/status_$tool.txt; exit 1; }
timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
  python -m pytest $SEL -q -x -p no:cacheprovider > $out/$tool.log 2>&1
echo "$tool rc=$?" > $out/status_$tool.txt

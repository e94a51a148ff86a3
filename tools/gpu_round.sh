#!/bin/bash
# One GPU call: smoke + gpu tests + bench (outputs under gpurun_out/)
tag=${1:-run}
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${tag}_tests.log
if [ "${2:-bench}" = "bench" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench=$?
  tail -c 1500 gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err
fi

set -x
AB_OUT=gpurun_out/conc_ab.jsonl AB_SET="0 1 0 1" VAR=OFSC_EXP_CONC timeout 900 tools/conc_ab.sh c4 c5
OFSC_TRACE=1 E2E_REPS=2 timeout 300 python tools/e2e_trace.py c4 > gpurun_out/e2e_trace.log 2>&1
OFSC_KMEANS_STATS=1 E2E_REPS=1 timeout 300 python tools/e2e_trace.py c4 > gpurun_out/km_stats.log 2>&1

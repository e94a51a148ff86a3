# SpMM static row assignment for L2-resident operands (OFSC_SPMM_STATIC_KB) at the small configs
for c in c1 c2 c3; do
VAR=OFSC_SPMM_STATIC_KB AB_SET="0 200000 0 200000" AB_OUT=gpurun_out/spmm_static_ab.jsonl ITER_METHODS=ofm_f2,ofm_f1 bash tools/conc_ab.sh $c > /dev/null
done
cat gpurun_out/spmm_static_ab.jsonl

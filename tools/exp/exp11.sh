for rep in 1 2; do for ip in 0 1; do
  OFSC_SPMM_IP=$ip python tools/spmm_time.py c4 c5 c6 c3 2>/dev/null | sed "s/^{/{\"ip\": $ip, /" >> gpurun_out/spmm_ip_ab.jsonl
done; done
for ip in 0 1; do OFSC_SPMM_IP=$ip ITER_METHODS=ofm_f2 ITER_TAG="ip=$ip" python tools/iter_time.py c4 >> gpurun_out/spmm_ip_iter.jsonl 2>/dev/null; done

# C2b fp64 with per-row TMA into the padded tiles, 2 CTAs/SM (OFSC_GS_PD=1) vs the warp-specialised copy kernel
VAR=OFSC_GS_PD AB_SET="0 1 0 1 0 1" AB_OUT=gpurun_out/gs_pd_ab.jsonl ITER_METHODS=ofm_f2,triofm_f2 bash tools/conc_ab.sh c4 c5 c3 > /dev/null
python - <<PY
import json, statistics as st
rows=[json.loads(l) for l in open("gpurun_out/gs_pd_ab.jsonl")]
for c in ("c4","c5","c3"):
  for m in ("ofm_f2","triofm_f2"):
    for v in ("0","1"):
        xs=[r["ms_per_iter"] for r in rows if r["config"]==c and r["method"]==m and r["tag"].endswith("="+v)]
        print(c, m, v, round(st.median(xs),4), [round(x,4) for x in xs])
PY
for v in 0 1; do OFSC_GS_PD=$v python - >> gpurun_out/gs_pd_kernel.jsonl 2>>gpurun_out/gs_pd_kernel.err <<'PY'
import sys, os, json
sys.path.insert(0, '.')
import torch, paper_2305_10356_b200 as ofsc
from synth import CONFIGS, config_graph, x0_block
cfg = CONFIGS["c4"]; s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
for rep in range(2):
    X = X0.clone(); r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
    print(json.dumps({"gs_pd": os.environ["OFSC_GS_PD"], "kernel_ms": [round(v / 10, 3) for v in r.report["kernel_ms"]], "checksum": float(X.double().sum())}), flush=True)
PY
done
cat gpurun_out/gs_pd_kernel.jsonl
OFSC_GS_PD=1 timeout 900 python -m pytest tests/test_gpu_iterate.py tests/test_gpu_kernels.py tests/test_gpu_multirank.py tests/test_gpu_rr.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2

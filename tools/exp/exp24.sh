# C3 (f2 methods): 8-row tiles x 4 stages (OFSC_C3_TR8=1) vs 16 x 2
VAR=OFSC_C3_TR8 AB_SET="0 1 0 1" AB_OUT=gpurun_out/c3_tr8_ab.jsonl ITER_METHODS=ofm_f2,triofm_f2 bash tools/conc_ab.sh c4 c5 c3 > /dev/null
cat gpurun_out/c3_tr8_ab.jsonl
for v in 0 1; do OFSC_C3_TR8=$v python - >> gpurun_out/c3_tr8_kernel.jsonl 2>>gpurun_out/c3_tr8_kernel.err <<'PY'
import sys, os, json
sys.path.insert(0, '.')
import torch, paper_2305_10356_b200 as ofsc
from synth import CONFIGS, config_graph, x0_block
cfg = CONFIGS["c4"]; s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
for rep in range(2):
    X = X0.clone(); r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
    print(json.dumps({"tr8": os.environ["OFSC_C3_TR8"], "kernel_ms": [round(v / 10, 3) for v in r.report["kernel_ms"]], "checksum": float(X.double().sum())}), flush=True)
PY
done
cat gpurun_out/c3_tr8_kernel.jsonl

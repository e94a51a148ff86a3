"""A/B the SpMM variants at a config (OFSC_SPMM_V = 1 | 2): per-launch ms and bitwise equality."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
ref = None
for v in ("1", "2", "1", "2"):
    os.environ["OFSC_SPMM_V"] = v
    X = X0.clone()
    r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
    if ref is None:
        ref = X.clone()
    print(json.dumps({"config": cfg.name, "v": v, "spmm_ms": r.report["kernel_ms"][3] / 10,
                      "bitwise_equal": bool(torch.equal(X, ref))}), flush=True)

"""Time the iteration at c4 for SpMM tuning knobs (env vars read per launch)."""
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
for ctas in ("2", "3", "4"):
    for ch in ("2", "4", "8", "16", "32"):
        os.environ["OFSC_SPMM_CTAS_PER_SM"] = ctas
        os.environ["OFSC_SPMM_CHUNK"] = ch
        X = X0.clone()
        r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
        print(json.dumps({"ctas": ctas, "chunk": ch, "spmm_ms": r.report["kernel_ms"][3] / 10,
                          "iter_ms": None}), flush=True)

"""Run T iterations of OFM-f2 on a config's reordered graph (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
method = sys.argv[3] if len(sys.argv) > 3 else "ofm_f2"
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
r = ofsc.run(g, method, X, T)
torch.cuda.synchronize()
print("done", r.report["iters"])

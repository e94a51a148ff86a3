"""c4 SpMM ms: L2 evict_first on the read-once streams (OFSC_SPMM_STREAM_HINT) A/B."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

cfg = CONFIGS["c4"]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
for rep in range(3):
    for sh in (0, 1):
        os.environ["OFSC_SPMM_STREAM_HINT"] = str(sh)
        X = X0.clone()
        r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
        km = r.report["kernel_ms"]
        print(json.dumps({"stream_hint": sh, "rep": rep, "spmm_ms": round(km[3] / 10, 4),
                          "gram_stream_ms": round(km[8] / 10, 4),
                          "iter_ms": round(sum(km) / 10, 4),
                          "checksum": float(X.double().sum())}), flush=True)

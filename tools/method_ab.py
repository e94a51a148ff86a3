"""Per-method C3 ms and graph-launched ms per iteration at the given configs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

for name in (sys.argv[1:] or ["c4"]):
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    for rep in range(2):
        for m in ofsc.METHODS:
            X = X0.clone()
            r = ofsc.run(g, m, X, 12, timing_skip=2, profile=True)
            km = r.report["kernel_ms"]
            X2 = X0.clone()
            r2 = ofsc.run(g, m, X2, 22, timing_skip=2)
            print(json.dumps({"config": name, "method": m, "rep": rep, "c3_ms": round(km[0] / 10, 4),
                              "graph_ms_per_iter": round(r2.report["timed_ms"] / 20, 4),
                              "checksum": float(X.double().sum())}), flush=True)
    g.close()

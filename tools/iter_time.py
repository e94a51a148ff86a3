"""Graph-launched ms per iteration (median of 3 runs of 20 timed iterations) per
method at the given configs; env switches are read once per process, so A/B runs
use one process per setting."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

methods = os.environ.get("ITER_METHODS", "ofm_f2,ofm_f1").split(",")
tag = os.environ.get("ITER_TAG", "")
for name in (sys.argv[1:] or ["c4"]):
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    for m in methods:
        ts = []
        for rep in range(3):
            X = X0.clone()
            r = ofsc.run(g, m, X, 22, timing_skip=2)
            ts.append(r.report["timed_ms"] / 20)
        ts.sort()
        print(json.dumps({"tag": tag, "config": name, "method": m, "ms_per_iter": round(ts[1], 4),
                          "all": [round(t, 4) for t in ts],
                          "checksum": float(X.double().sum())}), flush=True)
    g.close()

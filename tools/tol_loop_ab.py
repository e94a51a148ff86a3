"""Tolerance-mode run time: device-side while loop (OFSC_DEVLOOP=1) vs host polling."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    for rep in range(2):
        X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = ofsc.run(g, "ofm_f1", X, 2000, tol=1e-6, check_every=1)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t)
        print(json.dumps({"config": name, "devloop": os.environ.get("OFSC_DEVLOOP") == "1",
                          "iters": r.report["iters"], "converged": r.report["converged"],
                          "ms": round(ms, 2), "us_per_iter": round(1e3 * ms / max(r.report["iters"], 1), 2)}),
              flush=True)
    g.close()

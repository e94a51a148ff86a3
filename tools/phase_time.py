"""Per-phase kernel ms per iteration (profile mode, CUDA events) at the given configs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

NAMES = ["update_direction", "beta", "direction_gram", "spmm", "gram_reduce", "line_search",
         "comm", "refresh", "gram_stream", "unused"]
method = os.environ.get("METHOD", "ofm_f2")
for name in (sys.argv[1:] or ["c2"]):
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=cfg.n >= 100000)
    X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    r = ofsc.run(g, method, X, 42, timing_skip=2, profile=True)
    km = r.report["kernel_ms"]
    r2 = ofsc.run(g, method, torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda(), 42,
                  timing_skip=2)
    out = {"config": name, "method": method,
           "graph_ms_per_iter": r2.report["timed_ms"] / 40}
    out.update({n: round(km[i] / 40 * 1e3, 2) for i, n in enumerate(NAMES) if km[i] > 0})
    print(json.dumps(out), flush=True)
    g.close()

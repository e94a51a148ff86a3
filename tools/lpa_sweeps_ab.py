"""LPA sweep cap vs build time and SpMM time at a config (A/B of ofsc_build_opts.lpa_sweeps)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = CONFIGS[name]
s, d, _ = config_graph(cfg)
hs, hd = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
for rep in range(2):
    for sweeps in (4, 6, 10, 15, 30):
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = ofsc.Graph(cfg.n, hs, hd, reorder=True, lpa_sweeps=sweeps)
        torch.cuda.synchronize()
        build_ms = 1e3 * (time.perf_counter() - t)
        X = X0.clone()
        r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
        km = r.report["kernel_ms"]
        print(json.dumps({"config": name, "rep": rep, "sweeps": sweeps, "build_ms": round(build_ms, 2),
                          "communities": g.info["n_communities"],
                          "intra": round(g.info["intra_edge_fraction"], 4),
                          "spmm_ms": round(km[3] / 10, 4), "iter_ms": round(sum(km) / 10, 3)}),
              flush=True)
        g.close()

"""SpMM ms per launch vs the neighbour-scale stream (OFSC_SPMM_SVAL: 0 gathered s_j,
1 per-nonzero s_j, 2 packed column|degree + per-degree table), PF default rule."""
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
    X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    for rep in range(2):
        for mode in os.environ.get("MODES", "0,1,2").split(","):
            os.environ["OFSC_SPMM_SVAL"] = mode
            g = ofsc.Graph(cfg.n, s, d, reorder=True)
            X = X0.clone()
            r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
            km = r.report["kernel_ms"]
            print(json.dumps({"config": name, "sval_mode": int(mode), "rep": rep,
                              "max_degree": g.info["max_degree"],
                              "spmm_ms": round(km[3] / 10, 4), "iter_ms": round(sum(km) / 10, 4),
                              "checksum": float(X.double().sum())}), flush=True)
            g.close()
    os.environ.pop("OFSC_SPMM_SVAL", None)

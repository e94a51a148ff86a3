"""SpMM ms per launch vs the L2-prefetch variant (OFSC_SPMM_PF for graphs with the
s_j stream, OFSC_SPMM_PF_SMALL otherwise) at the given configs; one build per config."""
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
    big = g.info["nnz_global"] >= 20_000_000
    key = "OFSC_SPMM_PF" if big else "OFSC_SPMM_PF_SMALL"
    for rep in range(2):
        for pf in (0, 1, 2, 3):
            os.environ[key] = str(pf)
            X = X0.clone()
            r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
            km = r.report["kernel_ms"]
            print(json.dumps({"config": name, key: pf, "rep": rep,
                              "spmm_ms": round(km[3] / 10, 4), "iter_ms": round(sum(km) / 10, 4),
                              "checksum": float(X.double().sum())}), flush=True)
    os.environ.pop(key, None)
    g.close()

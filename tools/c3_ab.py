"""C3 (update + direction) ms per launch: k_update_direction vs a variant selected by
the environment variable VAR (default OFSC_C3_WS; round 2 also compared the removed
OFSC_C3_V2, profiles/r02/c3_v2_ab.jsonl); checksums must be identical (same bits)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

VAR = os.environ.get("VAR", "OFSC_C3_WS")

for name in (sys.argv[1:] or ["c4"]):
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    for rep in range(2):
        for m in ("ofm_f2", "ofm_f1", "triofm_f2"):
            for v in ("0", "1"):
                os.environ[VAR] = v
                X = X0.clone()
                r = ofsc.run(g, m, X, 12, timing_skip=2, profile=True)
                km = r.report["kernel_ms"]
                X2 = X0.clone()
                r2 = ofsc.run(g, m, X2, 22, timing_skip=2)
                print(json.dumps({"config": name, "method": m, VAR: int(v), "rep": rep,
                                  "c3_ms": round(km[0] / 10, 4), "c4_ms": round(km[2] / 10, 4),
                                  "c2b_ms": round(km[8] / 10, 4), "iter_ms": round(sum(km) / 10, 4),
                                  "graph_ms_per_iter": round(r2.report["timed_ms"] / 20, 4),
                                  "checksum": float(X.double().sum())}), flush=True)
    os.environ.pop(VAR, None)
    g.close()

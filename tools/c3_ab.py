"""C3 (update + direction) ms per launch: k_update_direction vs _v2 (OFSC_C3_V2),
# NOTE: the OFSC_C3_V2 variant this script compared was removed after the measurement (profiles/r02/c3_v2_ab.jsonl).
all four methods at the given configs; checksums must be identical (same bits)."""
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
        for m in ("ofm_f2", "ofm_f1"):
            for v in ("0", "1"):
                os.environ["OFSC_C3_V2"] = v
                X = X0.clone()
                r = ofsc.run(g, m, X, 12, timing_skip=2, profile=True)
                km = r.report["kernel_ms"]
                X2 = X0.clone()
                r2 = ofsc.run(g, m, X2, 22, timing_skip=2)
                print(json.dumps({"config": name, "method": m, "c3_v2": int(v), "rep": rep,
                                  "c3_ms": round(km[0] / 10, 4), "iter_ms": round(sum(km) / 10, 4),
                                  "graph_ms_per_iter": round(r2.report["timed_ms"] / 20, 4),
                                  "checksum": float(X.double().sum())}), flush=True)
    os.environ.pop("OFSC_C3_V2", None)
    g.close()

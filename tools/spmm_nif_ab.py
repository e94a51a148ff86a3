"""SpMM ms: 8 neighbour rows in flight at 3 CTAs/SM (80 registers) vs 6 at 4 CTAs/SM
(64 registers), OFSC_SPMM_NIF; same sums (CSR order), checksums must agree."""
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
    for rep in range(3):
        for nif in ("8", "6", "4"):
            os.environ["OFSC_SPMM_NIF"] = nif
            X = X0.clone()
            r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
            km = r.report["kernel_ms"]
            print(json.dumps({"config": name, "nif": int(nif), "rep": rep,
                              "spmm_ms": round(km[3] / 10, 4), "checksum": float(X.double().sum())}),
                  flush=True)
    os.environ.pop("OFSC_SPMM_NIF", None)
    g.close()

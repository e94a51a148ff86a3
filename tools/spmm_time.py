"""SpMM (C2a) ms per launch at the given configs (profiled run, CUDA events)."""
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
    X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
    km = r.report["kernel_ms"]
    print(json.dumps({"config": name, "spmm_ms": km[3] / 10, "gram_stream_ms": km[8] / 10,
                      "update_direction_ms": km[0] / 10, "direction_gram_ms": km[2] / 10,
                      "iter_ms": sum(km) / 10,
                      "checksum": float(X.double().sum())}), flush=True)
    g.close()

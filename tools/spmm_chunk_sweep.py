"""c4 SpMM ms vs rows per work grab (OFSC_SPMM_CHUNK) with the default stream/prefetch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
for rep in range(2):
    for ch in (2, 4, 6, 8, 16):
        os.environ["OFSC_SPMM_CHUNK"] = str(ch)
        X = X0.clone()
        r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
        km = r.report["kernel_ms"]
        print(json.dumps({"config": cfg.name, "chunk": ch, "rep": rep,
                          "spmm_ms": round(km[3] / 10, 4), "checksum": float(X.double().sum())}),
              flush=True)

"""One ofsc_spectral_cluster call at a config with OFSC_TRACE=1 phase timestamps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block, kmeans_init_rows  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
s, d, lab = config_graph(cfg)
X0 = x0_block(cfg.n, cfg.k, cfg.seed_x0)
rows = kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)
hs, hd = torch.from_numpy(s).pin_memory(), torch.from_numpy(d).pin_memory()
hx = torch.from_numpy(X0).pin_memory()
for rep in range(3):
    x = hx.clone().pin_memory()
    torch.cuda.synchronize()
    t = time.perf_counter()
    labels, feats, report = ofsc.spectral_cluster(cfg.n, hs.numpy(), hd.numpy(), "ofm_f2", x.numpy(),
                                                  cfg.blocks, rows, max_iters=cfg.iters)
    print(f"call {rep}: {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr, flush=True)

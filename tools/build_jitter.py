"""Graph build / append wall-clock jitter at c4 and c5 (repeated builds)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph  # noqa: E402

for name in sys.argv[1:] or ["c4"]:
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    for reorder in (False, True):
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t = time.perf_counter()
            g = ofsc.Graph(cfg.n, s, d, reorder=reorder)
            torch.cuda.synchronize()
            ts.append(round(1e3 * (time.perf_counter() - t), 1))
            g.close()
        print(name, "reorder" if reorder else "plain", "build ms", ts, flush=True)

"""Time ofsc.Graph builds at a config (reorder on / off), OFSC_TRACE=1 for phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
s, d, _ = config_graph(cfg)
hs, hd = torch.from_numpy(s).pin_memory(), torch.from_numpy(d).pin_memory()
for reorder in (True, False, True, False):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = ofsc.Graph(cfg.n, hs, hd, reorder=reorder)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    print(f"build reorder={reorder}: {ms:.1f} ms", file=sys.stderr, flush=True)
    g.close()

"""Time the K-means kernels at c4 scale (5M x 64 unit rows, K = 64) for a few Lloyd steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402

n, d, K = 5_000_000, 64, 64
g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
Y = ofsc.row_normalize(Y)
C0 = Y[:K].contiguous()
for steps in (1, 11):
    C = C0.clone()
    torch.cuda.synchronize()
    t = time.perf_counter()
    lab, it, inertia = ofsc.kmeans(Y, C, steps)
    torch.cuda.synchronize()
    print(f"steps={steps} iters={it} time={1e3 * (time.perf_counter() - t):.1f} ms", flush=True)

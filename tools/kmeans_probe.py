"""Time the K-means Lloyd step at c4 scale (5M x 64 unit rows, K = 64): fused
(assign + partial sums) vs the unfused kernels (OFSC_KMEANS_UNFUSED=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402

n, d, K = 5_000_000, 64, 64
g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
Y = ofsc.row_normalize(Y)
C0 = Y[:K].contiguous()
tag = "unfused" if os.environ.get("OFSC_KMEANS_UNFUSED") else "fused"
res = {}
for steps in (1, 1, 21, 41, 21, 41):
    C = C0.clone()
    torch.cuda.synchronize()
    t = time.perf_counter()
    lab, it, inertia = ofsc.kmeans(Y, C, steps)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    res.setdefault(steps, []).append(ms)
    print(f"{tag} steps={steps} iters={it} time={ms:.1f} ms "
          f"inertia={inertia:.12e} label_sum={int(lab.sum())}", flush=True)
print(f"{tag}: ms per Lloyd step = {(min(res[41]) - min(res[21])) / 20:.3f}")

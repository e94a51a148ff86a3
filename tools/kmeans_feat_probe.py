"""K-means on the pipeline's own features (config c3 or c4): build the graph,
run OFM-f2 for cfg.iters iterations, row-normalise, then time ofsc.kmeans from
the synth init rows.  OFSC_KMEANS_STATS=1 prints per-step skip statistics;
OFSC_KMEANS_NOSKIP=1 disables the bound test (A/B)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block, kmeans_init_rows  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = CONFIGS[name]
src, dst, lab = config_graph(cfg)
g = ofsc.Graph(cfg.n, torch.from_numpy(src), torch.from_numpy(dst), reorder=True)
X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
ofsc.run(g, "ofm_f2", X, cfg.iters)
Y = ofsc.row_normalize(X)
rows = torch.from_numpy(kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)).cuda()
for rep in range(3):
    C = Y[rows].double().contiguous()
    torch.cuda.synchronize()
    t = time.perf_counter()
    labels, it, inertia = ofsc.kmeans(Y, C, 100)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    print(f"{name} kmeans rep={rep} steps={it} ms={ms:.1f} per_step={ms / it:.3f} "
          f"inertia={inertia:.12e} label_sum={int(labels.sum())}", flush=True)
    os.environ.pop("OFSC_KMEANS_STATS", None)

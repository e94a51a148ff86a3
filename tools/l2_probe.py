"""L2 behaviour of the SpMM (C2a) on c4-shaped graphs: vary the within:between
ratio and the block-size law to separate intra-community capacity misses from
the random inter-community gathers.  Run under ncu (k_spmm DRAM bytes):
  VARIANT=intra python tools/l2_probe.py"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

VARIANTS = {
    "base": dict(),
    "intra": dict(ratio=1e6),
    "eq": dict(dirichlet=None),
    "intra_eq": dict(ratio=1e6, dirichlet=None),
    "small_blocks": dict(blocks=256),
}
v = os.environ.get("VARIANT", "base")
cfg = dataclasses.replace(CONFIGS["c4"], name="c4_" + v, **VARIANTS[v])
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
info = g.info
print(v, "communities", info["n_communities"], "intra", round(info["intra_edge_fraction"], 4), flush=True)
X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
r = ofsc.run(g, "ofm_f2", X, 4, timing_skip=1, profile=True)
print(v, "spmm_ms", r.report["kernel_ms"][3] / 3, flush=True)

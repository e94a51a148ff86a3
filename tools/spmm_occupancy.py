"""SpMM (C2a) ms per launch vs resident CTAs per SM and the L2 prefetch variant
(OFSC_SPMM_CTAS_PER_SM, OFSC_SPMM_PF), one graph build, profiled runs (CUDA events).
Question it answers: how much gather parallelism (warps per SM) the SpMM needs,
i.e. how many registers a fused SpMM + Gram kernel could give to DMMA warps."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = CONFIGS[name]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
grid = [(int(a), int(b)) for a, b in (x.split(":") for x in os.environ.get(
    "GRID", "3:0,3:1,3:2,3:0,3:1,3:2,2:0,2:2").split(","))]
for ctas, pf in grid:
    if True:
        os.environ["OFSC_SPMM_CTAS_PER_SM"] = str(ctas)
        os.environ["OFSC_SPMM_PF"] = str(pf)
        X = X0.clone()
        r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
        km = r.report["kernel_ms"]
        print(json.dumps({"config": name, "ctas_per_sm": ctas, "pf": pf,
                          "spmm_ms": round(km[3] / 10, 4), "iter_ms": round(sum(km) / 10, 4),
                          "checksum": float(X.double().sum())}), flush=True)
g.close()

"""Time the SpMM (C2a) at c4 for its tuning knobs (env vars read per launch):
OFSC_SPMM_CW (columns per pass), OFSC_SPMM_CHUNK (rows per work grab),
OFSC_SPMM_CTAS_PER_SM.  Usage: python tools/spmm_sweep.py [config] [--quick]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = CONFIGS[args[0] if args else "c4"]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d, reorder=True)
X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
ref = None
grid = [("64", "3", "8", h) for h in ("0", "1")] + [("32", "3", "8", h) for h in ("0", "1")]
if "--quick" not in sys.argv:
    grid += [("64", ct, ch, "1") for ct in ("2", "3", "4") for ch in ("4", "16")]
if "--default-hint" in sys.argv:                 # the production kernel (s_j stream, no hints)
    grid = [("64", ct, ch, "0") for ct in ("3", "4", "5") for ch in ("4", "8", "16", "32")]
for cw, ctas, ch, hint in grid:
    os.environ["OFSC_SPMM_HINT"] = hint
    os.environ["OFSC_SPMM_CW"] = cw
    os.environ["OFSC_SPMM_CTAS_PER_SM"] = ctas
    os.environ["OFSC_SPMM_CHUNK"] = ch
    X = X0.clone()
    r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, profile=True)
    if ref is None:
        ref = X.clone()
    err = float((X - ref).norm() / ref.norm())
    print(json.dumps({"hint": hint, "cw": cw, "ctas": ctas, "chunk": ch, "spmm_ms": r.report["kernel_ms"][3] / 10,
                      "iter_ms_total_profiled": sum(r.report["kernel_ms"]) / 10, "rel_diff_vs_first": err}),
          flush=True)

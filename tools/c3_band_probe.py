"""c3 (k = 64 inside a 71-eigenvalue cluster band): how many OFM iterations until
the features lie in span U_71 (sines) and how far span U_64 is resolved."""
import json
import os
import sys

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import eigsh

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402

cfg = CONFIGS["c3"]
s, d, _ = config_graph(cfg)
op = build_operator(cfg.n, s, d)
A = -sp.eye(cfg.n) - sp.diags(op.s) @ op.S @ sp.diags(op.s)
w, U = eigsh(A, k=73, which="SA", tol=1e-12)
i = np.argsort(w)
w, U = w[i], U[:, i]
g = ofsc.Graph(cfg.n, s, d, reorder=True)


def sines(Aa, B):
    qa, _ = np.linalg.qr(Aa)
    qb, _ = np.linalg.qr(B)
    return np.linalg.svd(qa - qb @ (qb.T @ qa), compute_uv=False)


for m in ("ofm_f1", "ofm_f2"):
    for T in (500, 1000, 2000, 4000, 8000):
        X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
        r = ofsc.run(g, m, X, T)
        Xh = X.cpu().numpy()
        print(json.dumps({"method": m, "T": T, "sin_band71": float(sines(Xh, U[:, :71]).max()),
                          "sin_U64": float(sines(Xh, U[:, :64]).max()),
                          "gnorm_ratio": r.report["grad_norm"] / r.report["grad_norm0"]}), flush=True)

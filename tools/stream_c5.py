#!/usr/bin/env python
"""Streaming protocol of BASELINE config c5.

N = 1M DCSBM graph (48 blocks, avg degree 16) revealed in 10 snapshots by
uniform edge sampling (10 % of the edges per stage).  Snapshot s is the union
of parts 1..s; its run is warm-started from the previous snapshot's features
(snapshot 1 from X0) and stops at ||G||_F <= tol * c_m * ||X||_F (R14), at most
`--max-iters` iterations.  Reports, per snapshot, the GPU graph build time, the
iterations to tolerance, the iteration time and the ARI of K-means (K = 48)
against the planted blocks; prints one JSON line.

  python tools/stream_c5.py [--method ofm_f1] [--tol 1e-4] [--parts 10] [--config c5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--method", default="ofm_f1")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--parts", type=int, default=10)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--paper-protocol", action="store_true",
                    help="fixed 2 iterations per stage (P:612) instead of the tolerance stop")
    ap.add_argument("--reorder", type=int, default=1)
    ap.add_argument("--sampling", default="edge", choices=["edge", "snowball"],
                    help="edge: uniform edge sampling (SGES); snowball: BFS-revealed edges "
                         "(SGSS, DESIGN.md R27); undiscovered nodes are isolated")
    ap.add_argument("--append", type=int, default=1,
                    help="1: ofsc_graph_append of each new part (incremental CSR merge, "
                         "NEXT-2); 0: rebuild each snapshot from the cumulative edge list")
    args = ap.parse_args()
    import torch
    import paper_2305_10356_b200 as ofsc
    from synth import CONFIGS, config_graph, stream_parts, snowball_parts, x0_block, kmeans_init_rows

    cfg = CONFIGS[args.config]
    src, dst, labels = config_graph(cfg)
    if args.sampling == "edge":
        parts = stream_parts(src, dst, args.parts, cfg.seed_graph + 1000)
    else:
        parts = snowball_parts(cfg.n, src, dst, args.parts, cfg.seed_graph + 2000)
    X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    rows = torch.from_numpy(kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)).cuda()
    stream = torch.cuda.current_stream()
    out = []
    cs, cd = [], []
    for si, (ps, pd) in enumerate(parts, 1):
        cs.append(ps)
        cd.append(pd)
        s = np.concatenate(cs)
        d = np.concatenate(cd)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        if args.append and si > 1:
            g.append(ps, pd)                 # incremental merge of part si (row order kept)
        else:
            if si > 1:
                g.close()
            g = ofsc.Graph(cfg.n, s, d, reorder=bool(args.reorder))
        b.record(stream)
        torch.cuda.synchronize()
        build_ms = a.elapsed_time(b)
        T = 2 if args.paper_protocol else args.max_iters
        tol = 0.0 if args.paper_protocol else args.tol
        r = ofsc.run(g, args.method, X, T, tol=tol, check_every=1, timing_skip=0)
        Y = ofsc.row_normalize(X)
        lab, km_it, _ = ofsc.kmeans(Y, Y[rows].contiguous(), 100)
        ari, nmi = ofsc.scores(lab.cpu().numpy(), labels)
        info = g.info
        out.append({"snapshot": si, "edges": int(s.size), "isolated": info["n_isolated"],
                    "build_ms": round(build_ms, 2), "iters": r.report["iters"],
                    "converged": r.report["converged"], "run_ms": round(r.report["timed_ms"], 2),
                    "ms_per_iter": round(r.report["timed_ms"] / max(r.report["iters"], 1), 3),
                    "grad_norm": r.report["grad_norm"], "ari": round(ari, 4), "nmi": round(nmi, 4)})
        print(json.dumps(out[-1]), file=sys.stderr, flush=True)
    g.close()
    print(json.dumps({"workload": f"{cfg.name} streaming, {args.parts} {args.sampling}-sampling snapshots",
                      "method": args.method, "tol": None if args.paper_protocol else args.tol,
                      "protocol": "2 its/stage (P:612)" if args.paper_protocol else "tolerance",
                      "reorder": bool(args.reorder),
                      "graph_update": "append (incremental CSR merge)" if args.append else "rebuild",
                      "total_iters": sum(o["iters"] for o in out),
                      "total_run_ms": round(sum(o["run_ms"] for o in out), 2),
                      "total_build_ms": round(sum(o["build_ms"] for o in out), 2),
                      "snapshots": out}))


if __name__ == "__main__":
    main()

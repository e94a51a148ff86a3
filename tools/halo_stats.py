"""Exchange volume of the halo layout at a config for p = 2, 4, 8 (local test
communicators on one GPU: graph build only).  Per rank: halo rows received and
own rows sent per exchange, vs the (p-1)/p * N rows of an all-gather."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
s, d, _ = config_graph(cfg)
for reorder in (False, True):
    for p in (2, 4, 8):
        halo, send, nl = [], [], []
        for r in range(p):
            comm = ofsc.LocalComm(p, r)
            g = ofsc.Graph(cfg.n, s, d, comm=comm, reorder=reorder)
            halo.append(g.info["halo_rows"])
            send.append(g.info["send_rows"])
            nl.append(g.n_local)
            g.close()
            comm.close()
        ag = (p - 1) * cfg.n / p
        print(json.dumps({"config": cfg.name, "reorder": reorder, "p": p,
                          "max_halo_rows": max(halo), "max_send_rows": max(send),
                          "allgather_rows_per_rank": int(ag),
                          "max_halo_over_allgather": round(max(halo) / ag, 3),
                          "bytes_per_exchange_max_rank": max(halo) * cfg.k * 8}), flush=True)

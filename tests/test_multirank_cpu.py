"""Multi-rank host logic on CPU (world_size 2, gloo): the library's nnz-balanced
row partition agrees across ranks and covers the graph, and the NCCL unique id
reaches every rank unchanged.  (The NCCL data path itself needs one GPU per
rank; its single-GPU layout is checked by tests/test_gpu_kernels.py with local
test communicators.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_10356_b200 as ofsc
        from oracle import build_operator
        from synth import CONFIGS, config_graph
        cfg = CONFIGS["c2"]
        s, d, _ = config_graph(cfg)
        op = build_operator(cfg.n, s, d)
        begins = ofsc.partition_rows(op.row_ptr, world)
        allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, torch.from_numpy(begins))
        same = all(torch.equal(allb[0], b) for b in allb)
        rb, re_ = int(begins[rank]), int(begins[rank + 1])
        nz = torch.tensor([int(op.row_ptr[re_] - op.row_ptr[rb]) + (re_ - rb)], dtype=torch.int64)
        dist.all_reduce(nz)
        uid = ofsc.Comm.broadcast_unique_id()
        uids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(uids, torch.tensor(list(uid), dtype=torch.uint8))
        q.put((rank, same, begins.tolist(), int(nz.item()), int(op.row_ptr[-1] + cfg.n),
               all(torch.equal(uids[0], u) for u in uids), len(uid)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e)))
    finally:
        dist.destroy_process_group()


def test_partition_and_unique_id_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    for rank, same, begins, nz_sum, nz_total, uid_same, uid_len in res:
        assert same and uid_same and uid_len == 128
        assert begins[0] == 0 and begins[-1] == 20_000 and begins[0] < begins[1] < begins[2]
        assert nz_sum == nz_total


def test_partition_balance_host():
    import paper_2305_10356_b200 as ofsc
    rng = np.random.default_rng(0)
    deg = rng.integers(0, 50, 10_000)
    rp = np.concatenate([[0], np.cumsum(deg)])
    for p in (1, 2, 3, 8):
        b = ofsc.partition_rows(rp, p)
        assert b[0] == 0 and b[-1] == 10_000 and np.all(np.diff(b) >= 0)
        w = np.array([rp[b[r + 1]] - rp[b[r]] + (b[r + 1] - b[r]) for r in range(p)])
        assert w.max() <= (rp[-1] + 10_000) / p + 51


# ---------------------------------------------------------------------------
# The p > 1 schedule on CPU ranks (gloo): rows split by the library's partition,
# each rank owns its rows of X, AX, G, V; per iteration it exchanges only the
# halo rows of V (the rows of its peers its columns reference; by symmetry of
# the graph, the rows it sends to q are its own rows with a neighbour in q's
# range -- the plan DESIGN.md sec. 8 derives without a handshake), sums its
# rows' Gram / column-dot partials over ranks in rank order (all-gather, then a
# fixed-order sum, as comm.cu does), and runs the replicated k x k line search.
# The result must equal the single-process oracle (Algorithm 2).
def _schedule_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_10356_b200 as ofsc
        from oracle import (build_operator, direction, cubic_coefficients, select_step,
                            objective, fro2_A)
        from synth import dcsbm_graph, x0_block
        n, k, T = 1500, 4, 6
        s, d, _ = dcsbm_graph(n, 5, 9000, 3.0, 31, 5.0)
        op = build_operator(n, s, d)
        b = ofsc.partition_rows(op.row_ptr, world)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        owner = np.searchsorted(b, np.arange(n), side="right") - 1
        S = op.S.tocsr()
        own_cols = S[r0:r1]
        # halo plan: receive from q the q-owned columns my rows reference (ascending);
        # send to q my rows that have a neighbour owned by q (ascending)
        cols = np.unique(own_cols.indices)
        recv = {qq: cols[owner[cols] == qq] for qq in range(world) if qq != rank}
        send = {}
        for qq in range(world):
            if qq == rank:
                continue
            rows = np.arange(r0, r1)
            has = np.array([np.any(owner[S.indices[S.indptr[i]:S.indptr[i + 1]]] == qq)
                            for i in rows], dtype=bool)
            send[qq] = rows[has]

        def exchange(Zloc):
            """Full-length buffer holding my rows and my halo (other rows NaN)."""
            buf = np.full((n, k), np.nan)
            buf[r0:r1] = Zloc
            reqs = []
            for qq, rows in send.items():
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(buf[rows])), qq))
            for qq, rows in recv.items():
                t = torch.empty((rows.size, k), dtype=torch.float64)
                dist.recv(t, qq)
                buf[rows] = t.numpy()
            for r_ in reqs:
                r_.wait()
            return buf

        def rank_sum(x):
            """all-gather of the rank partials, summed in rank order (comm.cu)."""
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            acc = parts[0].numpy().copy()
            for p_ in parts[1:]:
                acc = acc + p_.numpy()
            return acc

        sl = op.s[r0:r1, None]

        def apply_local(Zloc):
            buf = exchange(Zloc)
            nb = np.nan_to_num(buf) * op.s[:, None]          # unused (NaN) rows never referenced
            return -Zloc - sl * (own_cols @ nb)

        X0 = x0_block(n, k, 32)
        X = X0[r0:r1].copy()
        AX = apply_local(X)
        M, W = rank_sum(X.T @ X), rank_sum(X.T @ AX)
        Gp = Vp = ggp = None
        objs = []
        for t in range(T):
            G = direction("ofm_f2", X, AX, M, W)
            gg = rank_sum(np.sum(G * G, axis=0))
            objs.append(float(objective("ofm_f2", M, W, fro2_A(op))))
            if t == 0:
                V = -G
            else:
                num = rank_sum(np.sum((G - Gp) * G, axis=0))
                beta = np.maximum(np.where(ggp > 0, num / np.where(ggp > 0, ggp, 1), 0), 0)
                V = -G + Vp * beta[None, :]
            AV = apply_local(V)
            Q, P, Tm, Rp = (rank_sum(V.T @ V), rank_sum(V.T @ X), rank_sum(V.T @ AV),
                            rank_sum(X.T @ AV))
            a, _ = select_step(*[float(c) for c in cubic_coefficients("ofm_f2", Q, P, Tm, Rp, M, W)])
            X = X + a * V
            AX = AX + a * AV
            M = M + a * (P.T + P) + a * a * Q
            W = W + a * (Rp + Rp.T) + a * a * Tm
            Gp, Vp, ggp = G, V, gg
        parts = [torch.empty(n, k, dtype=torch.float64) for _ in range(world)]
        full = torch.zeros(n, k, dtype=torch.float64)
        full[r0:r1] = torch.from_numpy(X)
        dist.all_gather(parts, full)
        Xall = sum(p_.numpy() for p_ in parts)
        q.put((rank, Xall, objs, {qq: v.tolist() for qq, v in send.items()},
               {qq: v.tolist() for qq, v in recv.items()}))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_row_partitioned_schedule_two_ranks_matches_oracle():
    import torch.multiprocessing as mp
    from oracle import build_operator, run_ofm
    from synth import dcsbm_graph, x0_block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_schedule_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not isinstance(r[1], str), r[2]
    n, k = 1500, 4
    s, d, _ = dcsbm_graph(n, 5, 9000, 3.0, 31, 5.0)
    o = run_ofm(build_operator(n, s, d), "ofm_f2", x0_block(n, k, 32), 6, refresh=0)
    for rank, X, objs, send, recv in res:
        assert np.linalg.norm(X - o.X) / np.linalg.norm(o.X) <= 1e-12
        assert np.allclose(objs, o.history[:6, 0], rtol=1e-12, atol=0)
    # the exchange plan is symmetric: what 0 sends to 1 is exactly what 1 receives from 0
    assert res[0][3][1] == res[1][4][0] and res[1][3][0] == res[0][4][1]


def test_bench_launcher_spawns_ranks():
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks (one process
    per GPU, torch.distributed.run on 127.0.0.1); --dry-run makes each rank report."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1, 2]
    assert all(x["world"] == 3 and x["gpus"] == 3 for x in lines)
    # inside a launcher the world size must match --gpus
    env2 = dict(env, WORLD_SIZE="2", RANK="0")
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env2)
    assert bad.returncode != 0

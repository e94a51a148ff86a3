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

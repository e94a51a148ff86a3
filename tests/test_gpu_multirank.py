"""P5: the row-partitioned multi-GPU schedule at
p = 2, 3, 8 against the oracle and against p = 1.

One GPU is available per test box, so the p ranks run as an in-process local
world (ofsc_comm_create_local_world): one host thread per rank, each rank's
kernels on its own stream, the halo exchange and the sums over ranks carried
by host barriers + device copies.  Everything else -- nnz-balanced partition,
halo layout, packing, the split own-column / halo-column SpMM, the all-gather +
fixed rank-order sum of the Grams and column dots, beta, line search, the
K-means reductions -- is the code the NCCL run executes.
No kernel waits on another rank's kernel."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import (build_operator, kmeans_lloyd, row_normalize, run_ofm, METHODS)  # noqa: E402
from synth import CONFIGS, config_graph, kmeans_init_rows, x0_block  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


_C = {}


def c2():
    if "c2" not in _C:
        cfg = CONFIGS["c2"]
        s, d, lab = config_graph(cfg)
        _C["c2"] = (cfg, s, d, lab, build_operator(cfg.n, s, d), x0_block(cfg.n, cfg.k, cfg.seed_x0))
    return _C["c2"]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run_ranks(p, n, s, d, X0, method, T, reorder=False, dtype="f64", **kw):
    """Run `method` for T iterations on p local-world ranks; return the features
    in original node order (all rows), the per-rank reports and graph infos."""
    world = ofsc.LocalWorld(p)
    tdt = torch.float64 if dtype == "f64" else torch.float32

    def rank_fn(r, comm):
        g = ofsc.Graph(n, s, d, comm=comm, reorder=reorder)
        info = g.info
        perm = g.copy_perm()
        rows = perm[info["row_begin"]:info["row_end"]]
        X = torch.from_numpy(np.ascontiguousarray(X0[rows])).to(tdt).cuda()
        res = ofsc.run(g, method, X, T, debug=True, **kw)
        out = X.double().cpu().numpy()
        g.close()
        return rows, out, res, info

    try:
        outs = world.run(rank_fn)
    finally:
        world.close()
    Xf = np.zeros_like(X0, dtype=np.float64)
    for rows, out, _, _ in outs:
        Xf[rows] = out
    return Xf, [o[2] for o in outs], [o[3] for o in outs]


@pytest.mark.parametrize("p", [2, 3, 8])
@pytest.mark.parametrize("method", METHODS)
def test_p5_ten_steps_vs_oracle(p, method):
    """North-star tolerance at p ranks: 10 iterations, rel. Frobenius <= 1e-10 vs the oracle."""
    cfg, s, d, lab, op, X0 = c2()
    o = run_ofm(op, method, X0, 10, refresh=0)
    Xp, reps, infos = run_ranks(p, cfg.n, s, d, X0, method, 10)
    assert all(r.report["iters"] == 10 for r in reps)
    # every rank took the same steps (replicated k x k state)
    for r in reps[1:]:
        assert np.array_equal(r.alphas, reps[0].alphas)
        assert np.array_equal(r.codes, reps[0].codes)
    assert rel(Xp, o.X) <= 1e-10
    assert np.allclose(reps[0].history[:, :2], o.history[:, :2], rtol=1e-9, atol=0)
    # the partition covers the rows once, balanced by nnz
    bounds = sorted((i["row_begin"], i["row_end"]) for i in infos)
    assert bounds[0][0] == 0 and bounds[-1][1] == cfg.n
    assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
    assert infos[0]["load_imbalance"] < 1.05


@pytest.mark.parametrize("p", [2, 8])
@pytest.mark.parametrize("method", ["ofm_f2", "triofm_f1"])
def test_p5_reordered_graph(p, method):
    """LPA locality order (communities stay on one rank): same mathematics (R23)."""
    cfg, s, d, lab, op, X0 = c2()
    o = run_ofm(op, method, X0, 10, refresh=0)
    Xp, reps, infos = run_ranks(p, cfg.n, s, d, X0, method, 10, reorder=True)
    assert all(i["reordered"] == 1 for i in infos)
    assert rel(Xp, o.X) <= 1e-10


@pytest.mark.parametrize("p", [2, 3])
def test_p5_paper_schedule_refresh(p):
    """refresh = 1 (AX recomputed every iteration): the X halo exchange too."""
    cfg, s, d, lab, op, X0 = c2()
    o = run_ofm(op, "ofm_f1", X0, 10, refresh=1)
    Xp, reps, _ = run_ranks(p, cfg.n, s, d, X0, "ofm_f1", 10, refresh=1)
    assert rel(Xp, o.X) <= 1e-10


def test_p5_matches_single_gpu_and_is_deterministic():
    """p = 3 vs p = 1 (both on the device): rounding-level agreement; p = 3 twice:
    bitwise identical (fixed rank-order sums, fixed per-CTA partial order)."""
    cfg, s, d, lab, op, X0 = c2()
    g = ofsc.Graph(cfg.n, s, d)
    X1 = torch.from_numpy(X0.copy()).cuda()
    ofsc.run(g, "ofm_f2", X1, 10)
    X1 = X1.cpu().numpy()
    a, _, _ = run_ranks(3, cfg.n, s, d, X0, "ofm_f2", 10)
    b, _, _ = run_ranks(3, cfg.n, s, d, X0, "ofm_f2", 10)
    assert np.array_equal(a, b)
    assert rel(a, X1) <= 1e-11


def test_p5_fp32():
    """fp32 storage at p = 2 vs the precision-matched oracle (P2 fp32 tolerance)."""
    cfg, s, d, lab, op, X0 = c2()
    X0r = X0.astype(np.float32).astype(np.float64)
    o = run_ofm(op, "ofm_f2", X0r, 10, refresh=0, precision="f32")
    Xp, _, _ = run_ranks(2, cfg.n, s, d, X0r, "ofm_f2", 10, dtype="f32")
    assert rel(Xp, o.X) <= 1e-4


@pytest.mark.parametrize("p", [2, 8])
def test_p5_kmeans_labels_equal_single_rank(p, capfd, monkeypatch):
    """K-means at p ranks on identical features: labels equal the oracle's Lloyd run
    (and therefore p = 1's, tested in test_gpu_cluster.py), ties excepted; the
    late steps run as light steps (bounds first, sums by label changes, the
    change sums and counts summed over ranks)."""
    monkeypatch.setenv("OFSC_KMEANS_STATS", "1")
    cfg, s, d, lab, op, X0 = c2()
    o = run_ofm(op, "ofm_f2", X0, 60, refresh=0)
    Y = row_normalize(o.X)
    K = cfg.blocks
    init = kmeans_init_rows(cfg.n, K, cfg.seed_km)
    C0 = Y[init].copy()
    lab_o, C_o, it_o, inertia_o = kmeans_lloyd(Y, C0, 100)
    bounds = np.linspace(0, cfg.n, p + 1).astype(np.int64)
    world = ofsc.LocalWorld(p)

    def rank_fn(r, comm):
        Yr = torch.from_numpy(np.ascontiguousarray(Y[bounds[r]:bounds[r + 1]])).cuda()
        C = torch.from_numpy(C0.copy()).cuda()
        labels, it, inertia = ofsc.kmeans(Yr, C, 100, comm=comm)
        return labels.cpu().numpy(), it, inertia, C.cpu().numpy()

    try:
        outs = world.run(rank_fn)
    finally:
        world.close()
    labels = np.concatenate([o_[0] for o_ in outs])
    steps = [l for l in capfd.readouterr().err.splitlines() if "[ofsc kmeans]" in l]
    assert len(steps) == p * outs[0][1] and sum(l.endswith("light 1") for l in steps) >= p
    assert all(o_[1] == outs[0][1] for o_ in outs)
    assert all(np.array_equal(o_[3], outs[0][3]) for o_ in outs)   # replicated centroids
    mism = np.nonzero(labels != lab_o)[0]
    assert mism.size <= 2, mism
    assert abs(outs[0][2] - inertia_o) <= 1e-9 * inertia_o
    assert np.allclose(outs[0][3], C_o, rtol=0, atol=1e-12)


def test_p5_spectral_cluster_end_to_end():
    """Algorithm 1 from host buffers at p = 2 (each rank fills its own nodes) vs p = 1."""
    cfg, s, d, lab, op, X0 = c2()
    init = kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)
    l1, F1, _ = ofsc.spectral_cluster(cfg.n, s, d, "ofm_f2", X0, cfg.blocks, init, max_iters=40,
                                      reorder=False)
    world = ofsc.LocalWorld(2)

    def rank_fn(r, comm):
        return ofsc.spectral_cluster(cfg.n, s, d, "ofm_f2", X0, cfg.blocks, init, max_iters=40,
                                     reorder=False, comm=comm,
                                     stream=torch.cuda.current_stream())

    try:
        outs = world.run(rank_fn)
    finally:
        world.close()
    labels = np.full(cfg.n, -1, np.int32)
    F = np.zeros_like(F1)
    for lr, Fr, _ in outs:
        own = lr >= 0
        labels[own] = lr[own]
        F[own] = Fr[own]
    assert np.all(labels >= 0)
    assert rel(F, F1) <= 1e-9
    ari, _ = ofsc.scores(labels, l1)
    assert ari >= 0.999


def test_local_world_missing_rank_fails_instead_of_hanging(monkeypatch):
    """A rank that never reaches a collective (here rank 1 makes no call) must not
    hang the others forever: the barrier wait is bounded (OFSC_LOCAL_WORLD_TIMEOUT_S)
    and the call fails with OFSC_ERR_STATE; the world stays failed afterwards."""
    monkeypatch.setenv("OFSC_LOCAL_WORLD_TIMEOUT_S", "2")
    cfg, s, d, lab, op, X0 = c2()
    Y = torch.from_numpy(np.ascontiguousarray(X0[:1000])).cuda()
    world = ofsc.LocalWorld(2)

    def rank_fn(r, comm):
        if r == 1:
            return None
        C = Y[:4].clone().contiguous()
        with pytest.raises(ofsc.OfscError) as e:
            ofsc.kmeans(Y, C, 5, comm=comm)
        assert e.value.status == 7
        with pytest.raises(ofsc.OfscError):
            ofsc.kmeans(Y, C, 5, comm=comm)
        return "failed as expected"

    try:
        out = world.run(rank_fn, timeout=120)
    finally:
        world.close()
    assert out[0] == "failed as expected"

"""Iteration parity: P1 (one step), P2 (10-step trajectory), P3 invariants.

The CUDA path runs Algorithm 2 through ofsc_run (C ABI); the oracle runs the
same schedule in numpy from the same seeded X0."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator, run_ofm, dense_A, METHODS, jacobi_eigh  # noqa: E402
from synth import CONFIGS, config_graph, x0_block, dcsbm_graph  # noqa: E402
from tests import graphs as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


_CACHE = {}


def setup(name):
    if name not in _CACHE:
        cfg = CONFIGS[name]
        s, d, lab = config_graph(cfg)
        op = build_operator(cfg.n, s, d)
        g = ofsc.Graph(cfg.n, s, d)
        X0 = x0_block(cfg.n, cfg.k, cfg.seed_x0)
        _CACHE[name] = (cfg, op, g, X0, lab)
    return _CACHE[name]


def gpu_run(g, method, X0, T, dtype="f64", **kw):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.from_numpy(np.array(X0)).to(tdt).cuda()
    r = ofsc.run(g, method, X, T, debug=True, **kw)
    return X.double().cpu().numpy(), r


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("refresh", [0, 1])
def test_p1_one_step(name, method, refresh):
    cfg, op, g, X0, _ = setup(name)
    o = run_ofm(op, method, X0, 1, refresh=refresh)
    X, r = gpu_run(g, method, X0, 1, refresh=refresh)
    assert r.report["iters"] == 1
    assert rel(X, o.X) <= 1e-12
    assert list(r.codes[0]) == list(o.codes[0])
    assert np.max(np.abs(r.alphas[0] - o.alphas[0])) <= 1e-12 * np.max(np.abs(o.alphas[0]))
    assert abs(r.history[0, 0] - o.history[0, 0]) <= 1e-12 * abs(o.history[0, 0])


@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("refresh", [0, 1])
def test_p2_ten_steps(name, method, refresh):
    """North-star tolerance: relative Frobenius error <= 1e-10 after 10 iterations (fp64)."""
    cfg, op, g, X0, _ = setup(name)
    o = run_ofm(op, method, X0, 10, refresh=refresh)
    X, r = gpu_run(g, method, X0, 10, refresh=refresh)
    assert r.report["iters"] == o.iters == 10
    first_flip = next((t for t in range(10) if list(r.codes[t]) != list(o.codes[t])), None)
    assert rel(X, o.X) <= 1e-10, f"branch codes first differ at t={first_flip}"
    assert np.allclose(r.history[:, :2], o.history[:, :2], rtol=1e-9, atol=0)


@pytest.mark.parametrize("method", METHODS)
def test_p2_fp32_against_precision_matched_oracle(method):
    cfg, op, g, X0, _ = setup("c2")
    X0r = X0.astype(np.float32).astype(np.float64)
    o = run_ofm(op, method, X0r, 10, refresh=0, precision="f32")
    X, r = gpu_run(g, method, X0r, 10, dtype="f32", refresh=0)
    assert rel(X, o.X) <= 1e-4


@pytest.mark.parametrize("method", METHODS)
def test_other_options(method):
    cfg, op, g, X0, _ = setup("c1")
    for kw in ({"beta_rule": "pr"}, {"beta_rule": "zero"}, {"refresh": 3},
               {"line_search": False, "alpha_fixed": 0.05, "beta_rule": "zero"}):
        o = run_ofm(op, method, X0, 8, **kw)
        X, r = gpu_run(g, method, X0, 8, **kw)
        assert rel(X, o.X) <= 1e-10, kw


def test_tolerance_stop_and_zero_start():
    cfg, op, g, X0, _ = setup("c1")
    o = run_ofm(op, "ofm_f1", X0, 400, tol=1e-6)
    X, r = gpu_run(g, "ofm_f1", X0, 400, tol=1e-6, check_every=4)
    assert r.report["converged"] == 1 and o.converged
    assert r.report["iters"] == o.iters
    assert rel(X, o.X) <= 1e-8
    X, r = gpu_run(g, "ofm_f2", np.zeros_like(X0), 5)
    assert r.report["converged"] == 1 and r.report["iters"] == 0 and np.all(X == 0)


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_p3_subspace_c1(method):
    """Converged OFM features span the bottom-k eigenvectors (sines <= 1e-6), and
    the GPU objective matches the oracle's at the config length."""
    cfg, op, g, X0, _ = setup("c1")
    w, U = np.linalg.eigh(dense_A(op))
    X, r = gpu_run(g, method, X0, cfg.iters)
    o = run_ofm(op, method, X0, cfg.iters, refresh=0)
    qa, _ = np.linalg.qr(X)
    c = np.linalg.svd(qa.T @ U[:, :cfg.k], compute_uv=False)
    assert np.sqrt(np.clip(1 - c ** 2, 0, 1)).max() <= 1e-6
    f_gpu, f_or = r.history[-1, 0], o.history[-1, 0]
    assert abs(f_gpu - f_or) <= 1e-10 * abs(f_or)


def test_p3_triofm_ordered_fixed_points():
    """Theorems 2/4 on a well-separated spectrum (bridged cliques): ordered columns."""
    pairs, n = G.bridged_cliques([5, 7, 9, 12], bridges=3)
    s, d = G.edges(pairs)
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d)
    w, U = jacobi_eigh(dense_A(op))
    X0 = x0_block(n, 4, 7)
    X, r = gpu_run(g, "triofm_f1", X0, 3000, beta_rule="pr")
    assert np.allclose(np.diag(X.T @ X), -w[:4], atol=1e-8)
    X, r = gpu_run(g, "triofm_f2", X0, 3000)
    assert np.allclose(X.T @ X, np.eye(4), atol=1e-8)


def test_divergence_reports_last_finite_iterate():
    cfg, op, g, X0, _ = setup("c1")
    Xbig = X0 * 1e200                  # squares overflow: non-finite direction at t = 0
    X = torch.from_numpy(Xbig).cuda()
    r = ofsc.run(g, "ofm_f1", X, 5, raise_on_diverge=False)
    assert r.report["diverged"] == 1 and r.report["iters"] == 0
    assert np.array_equal(X.cpu().numpy(), Xbig)
    with pytest.raises(ofsc.OfscDiverged):
        ofsc.run(g, "ofm_f1", torch.from_numpy(Xbig).cuda(), 5)


def test_warm_start_continues_trajectory():
    """Running 6 then 4 more iterations from the returned X equals a restart of CG
    (beta = 0 at the restart) in the oracle as well."""
    cfg, op, g, X0, _ = setup("c1")
    X, _ = gpu_run(g, "ofm_f2", X0, 6)
    X2, _ = gpu_run(g, "ofm_f2", X, 4)
    o1 = run_ofm(op, "ofm_f2", X0, 6, refresh=0)
    o2 = run_ofm(op, "ofm_f2", o1.X, 4, refresh=0)
    assert rel(X2, o2.X) <= 1e-10


def test_full_size_c4_sampled_rows():
    """BASELINE c4 (N = 5M, 50M edges, k = 64) at full size: the fused SpMM + Gram
    output on 2000 sampled rows against a row-by-row oracle, and the Grams
    against properties that hold at any size (symmetry of Z^T Z, trace identity)."""
    cfg = CONFIGS["c4"]
    s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d)
    assert g.info["n_edges_kept"] == cfg.edges
    rng = np.random.default_rng(0)
    torch.manual_seed(0)
    Z = torch.randn(cfg.n, 64, dtype=torch.float64, device="cuda") / np.sqrt(cfg.n)
    X = torch.randn(cfg.n, 64, dtype=torch.float64, device="cuda") / np.sqrt(cfg.n)
    Y, Gm = g.apply_gram(Z, X)
    rows = np.sort(rng.choice(cfg.n, 2000, replace=False))
    rp, col, sv = g.copy_csr()
    # oracle per row: canonical neighbour set from the raw edge list
    keep = s != d
    u, v = np.minimum(s[keep], d[keep]), np.maximum(s[keep], d[keep])
    key = np.sort(u * cfg.n + v)
    key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    uu, vv = key // cfg.n, key % cfg.n
    deg = np.bincount(np.concatenate([uu, vv]), minlength=cfg.n)
    nb = {r: [] for r in rows.tolist()}
    m1, m2 = np.isin(uu, rows), np.isin(vv, rows)
    for a, b in zip(uu[m1], vv[m1]):
        nb[a].append(b)
    for a, b in zip(vv[m2], uu[m2]):
        nb[a].append(b)
    Zh = Z.cpu().numpy()
    Yh = Y.cpu().numpy()
    for r in rows[:300]:
        js = np.array(sorted(nb[r]), dtype=np.int64)
        assert len(js) == deg[r] == rp[r + 1] - rp[r]
        sj = 1.0 / np.sqrt(deg[js])
        si = 1.0 / np.sqrt(deg[r]) if deg[r] else 0.0
        want = -Zh[r] - si * (sj[:, None] * Zh[js]).sum(0)
        assert np.max(np.abs(Yh[r] - want)) <= 1e-13 * max(1e-300, np.max(np.abs(want)))
    Gh = Gm.cpu().numpy()
    assert np.max(np.abs(Gh[0] - Gh[0].T)) <= 1e-14 * np.max(np.abs(Gh[0]))
    # tr(Z^T Y) = sum_i <Z_i, Y_i> (any size): check against a fp64 torch reduction
    assert abs(np.trace(Gh[2]) - float((Z * Y).sum())) <= 1e-10 * abs(np.trace(Gh[2]))


@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("method", METHODS)
def test_p2_reordered_graph(name, method):
    """The locality-reordered operator P A P^T gives the same iterates (rows mapped
    back to the original order by the library) within the north-star tolerance."""
    cfg, op, g, X0, _ = setup(name)
    gr = ofsc.Graph(cfg.n, *config_graph(cfg)[:2], reorder=True)
    o = run_ofm(op, method, X0, 10, refresh=0)
    X, r = gpu_run(gr, method, X0, 10)
    assert rel(X, o.X) <= 1e-10


_WIDE = {}


def setup_wide(k):
    """c3-shaped DCSBM at a ragged N = 20,011 for the KP = 48 / 64 kernels
    (symmetric DMMA Grams, register-resident M/W fragments), k = 48 or 64."""
    if k not in _WIDE:
        n = 20_011
        s, d, _ = dcsbm_graph(n, 24, 160_000, 3.0, 401 + k, 5.0)
        op = build_operator(n, s, d)
        g = ofsc.Graph(n, s, d, reorder=True)
        X0 = x0_block(n, k, 402 + k)
        _WIDE[k] = (op, g, X0)
    return _WIDE[k]


@pytest.mark.parametrize("k", [48, 64])
@pytest.mark.parametrize("method", METHODS)
def test_p2_wide_kernels(k, method):
    """P1 + P2 on the padded widths of the production configs (c3/c4: k = 64,
    c5: k = 48), reordered graph as in bench.py: one step 1e-12 with identical
    branch codes, ten steps 1e-10 (north-star tolerance)."""
    op, g, X0 = setup_wide(k)
    o1 = run_ofm(op, method, X0, 1, refresh=0)
    X1, r1 = gpu_run(g, method, X0, 1)
    assert rel(X1, o1.X) <= 1e-12
    assert list(r1.codes[0]) == list(o1.codes[0])
    o = run_ofm(op, method, X0, 10, refresh=0)
    X, r = gpu_run(g, method, X0, 10)
    assert rel(X, o.X) <= 1e-10
    assert np.allclose(r.history[:, :2], o.history[:, :2], rtol=1e-9, atol=0)


def _degenerate_cases():
    rng = np.random.default_rng(21)
    cases = {
        "no_edges_A_is_minus_I": (50, np.array([], np.int64), np.array([], np.int64), 4),
        "messy_k_equals_n": (12,) + GRAPHS_MESSY + (12,),
        "single_node": (1, np.array([], np.int64), np.array([], np.int64), 1),
        "star_bipartite": (9,) + G.edges(G.star(8)) + (3,),
        "two_cliques_k2": (14,) + G.edges(G.clique_union([8, 6])[0]) + (2,),
        "sparse_isolated": (400, rng.integers(0, 400, 120), rng.integers(0, 400, 120), 6),
    }
    return cases


GRAPHS_MESSY = (np.array([0, 1, 1, 2, 3, 3, 5, 9, 9, 7]), np.array([1, 0, 1, 3, 2, 2, 5, 8, 7, 9]))


@pytest.mark.parametrize("case", list(_degenerate_cases()))
@pytest.mark.parametrize("method", METHODS)
def test_degenerate_graphs(case, method):
    """Degenerate inputs of the method: no edges (A = -I, one repeated
    eigenvalue), k = n with self-loops / duplicates / isolated nodes, a single
    node, a bipartite star (eigenvalue 0 of A), a clique union with k equal to
    the number of components, a mostly isolated sparse graph: 10 iterations
    match the oracle (same iteration count, 1e-10 relative, or both diverge /
    stop at the same step)."""
    n, s, d, k = _degenerate_cases()[case]
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d)
    X0 = x0_block(n, k, 77) * np.sqrt(n)                 # O(1) entries on tiny graphs
    o = run_ofm(op, method, X0, 10, refresh=0)
    X, r = gpu_run(g, method, X0, 10)
    assert r.report["iters"] == o.iters
    assert bool(r.report["converged"]) == bool(o.converged)
    if rel(X, o.X) > 1e-10:
        # Several results are correct (R22): on a fully degenerate spectrum (A = -I)
        # TriOFM's per-column cubics have mirror-image roots whose psi values tie
        # to rounding, so the two sides may take different (equally good) roots.
        # Then the first differing step must be such a three-root choice with
        # equal psi, and both trajectories must reach the unique minimum: for A = -I
        # f1* = sum_{i>k} lambda_i^2 = n - k (Theorem 2's fixed points; pinned in
        # test_oracle_methods) and f2* = sum_{i<=k} lambda_i = -k.  After a different
        # root the two approach it at different rates (measured 1.4e-9 vs 1.8e-6
        # from f1* = 46 after 10 iterations), so they are compared with the limit,
        # not with each other.
        t = next(t for t in range(o.iters) if list(r.codes[t]) != list(o.codes[t])
                 or np.max(np.abs(r.alphas[t] - o.alphas[t])) > 1e-9 * np.max(np.abs(o.alphas[t])))
        assert method.startswith("tri") and case == "no_edges_A_is_minus_I", (case, method, t)
        assert any(8 <= c <= 10 for c in o.codes[t]), o.codes[t]
        fstar = float(n - k) if method.endswith("f1") else -float(k)
        for f in (o.history[-1, 0], r.history[-1, 0]):
            assert abs(f - fstar) <= 1e-6 * abs(fstar), (f, fstar)
    g.close()


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("method", ["ofm_f2", "triofm_f1"])
def test_streamed_neighbour_scales_bitwise(method, mode, monkeypatch):
    """The neighbour-scale streams (on by default for graphs with > 2e7 nonzeros,
    forced here on c2): per-nonzero s_j (mode 1) and the packed (column | degree)
    stream with a per-degree s table (mode 2) compute exactly the same sums as the
    gathered s_j."""
    cfg, op, g, X0, _ = setup("c2")
    X_a, _ = gpu_run(g, method, X0, 10)
    monkeypatch.setenv("OFSC_SPMM_SVAL", mode)
    s, d, _ = config_graph(cfg)
    g2 = ofsc.Graph(cfg.n, s, d)
    X_b, _ = gpu_run(g2, method, X0, 10)
    assert np.array_equal(X_a, X_b)
    o = run_ofm(op, method, X0, 10, refresh=0)
    assert rel(X_b, o.X) <= 1e-10
    g2.close()


@pytest.mark.parametrize("method", METHODS)
def test_graph_launch_structure_is_transparent(method):
    """The captured iteration (Q/P reduction on a forked branch, T/R' reduction fused
    with the line search in its last CTA) and the per-launch profiled sequence
    (separate reductions and line search on one stream) compute the same numbers
    bit for bit: identical reductions, identical line search."""
    cfg, op, g, X0, _ = setup("c2")
    Xa, ra = gpu_run(g, method, X0, 25)
    Xb, rb = gpu_run(g, method, X0, 25, profile=True)
    assert np.array_equal(Xa, Xb)
    assert np.array_equal(ra.history, rb.history)


@pytest.mark.parametrize("k", [48, 64])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("method", METHODS)
def test_c3_kernel_variants_bitwise(method, dtype, k, monkeypatch):
    """C3's two kernels -- the single-role k_update_direction and the producer-warp
    k_update_direction_ws (default for the f1 methods) -- compute the same bits
    (same products, same k order, explicitly rounded G expression; only the TMA
    traffic is owned differently), on the KP = 48 / 64 production widths
    (reordered N = 20,011 graph).  Both run the same grid: the column-dot
    partials, and so beta, depend on which tiles a CTA owns."""
    op, g, X0 = setup_wide(k)
    outs = []
    for ws, tr8 in (("0", "0"), ("1", "0"), ("0", "1")):   # + the 8-row x 4-stage form
        monkeypatch.setenv("OFSC_C3_WS", ws)
        monkeypatch.setenv("OFSC_C3_TR8", tr8)
        X, r = gpu_run(g, method, X0, 10, dtype=dtype)
        outs.append((X, r.history))
    for X, h in outs[1:]:
        assert np.array_equal(outs[0][0], X)
        assert np.array_equal(outs[0][1], h)

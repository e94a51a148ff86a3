"""Parity at the production configs (north_star: "all four methods
match the CPU oracle ... on every config").

  P2  c3 (N = 200k, k = 64, reordered as bench.py runs it): 10 iterations, all four
      methods, <= 1e-10 relative Frobenius (north-star fp64 tolerance).
  P2  c2 with the literal Polak-Ribiere rule of Alg. 2 l.9 (no clamp).
  P1+ c4 (N = 5M, E = 50M, k = 64) at full size: 2 iterations of every method
      (branch codes identical, alpha 1e-12, X 1e-12); fp32 storage at c4 against
      the precision-matched oracle (5 iterations, P2 fp32 tolerance 1e-4).
  P3  c2 at its config length (500 iterations): OFM-f1/f2 features span the exact
      bottom-32 eigenvectors (scipy eigsh, test-side library check) to sines
      <= 1e-6 and agree with the oracle's; the c3 shape with 64 planted blocks
      (separated lambda_64 / lambda_65) reaches span U_64 to 1e-6; c3 itself
      (lambda_64, lambda_65 2e-4 apart inside a 71-eigenvalue band) does not in
      any feasible run, so there the monotone objective, the approach to the
      band and the Ritz values inside it are asserted.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import scipy.sparse as sp  # noqa: E402
from scipy.sparse.linalg import eigsh  # noqa: E402

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator, run_ofm, METHODS  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


_C = {}


def setup(name, reorder):
    key = (name, reorder)
    if key not in _C:
        cfg = CONFIGS[name]
        s, d, lab = config_graph(cfg)
        op = _C.get(("op", name)) or build_operator(cfg.n, s, d)
        _C[("op", name)] = op
        g = ofsc.Graph(cfg.n, s, d, reorder=reorder)
        _C[key] = (cfg, op, g, x0_block(cfg.n, cfg.k, cfg.seed_x0))
    return _C[key]


def gpu_run(g, method, X0, T, dtype="f64", **kw):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.from_numpy(np.array(X0)).to(tdt).cuda()
    r = ofsc.run(g, method, X, T, debug=True, **kw)
    return X.double().cpu().numpy(), r


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def sines(A, B):
    """Principal-angle sines between span(A) and span(B), dim A <= dim B:
    singular values of (I - Qb Qb^T) Qa (accurate for small angles)."""
    qa, _ = np.linalg.qr(A)
    qb, _ = np.linalg.qr(B)
    return np.linalg.svd(qa - qb @ (qb.T @ qa), compute_uv=False)


def bottom_eigs(op, k):
    """Test-side library check: scipy eigsh on A = -I - D^{-1/2} S D^{-1/2}."""
    Sn = sp.diags(op.s) @ op.S @ sp.diags(op.s)
    A = -sp.eye(op.n) - Sn
    w, U = eigsh(A, k=k, which="SA", tol=1e-12)
    i = np.argsort(w)
    return w[i], U[:, i]


@pytest.mark.parametrize("method", METHODS)
def test_p2_c3_ten_steps(method):
    cfg, op, g, X0 = setup("c3", True)
    o = run_ofm(op, method, X0, 10, refresh=0)
    X, r = gpu_run(g, method, X0, 10)
    assert r.report["iters"] == o.iters == 10
    first_flip = next((t for t in range(10) if list(r.codes[t]) != list(o.codes[t])), None)
    assert rel(X, o.X) <= 1e-10, f"branch codes first differ at t={first_flip}"
    assert np.allclose(r.history[:, :2], o.history[:, :2], rtol=1e-9, atol=0)


@pytest.mark.parametrize("method", METHODS)
def test_p2_c2_literal_polak_ribiere(method):
    """beta_rule = "pr": the printed column-wise formula of Alg. 2 l.9 without the PR+ clamp."""
    cfg, op, g, X0 = setup("c2", False)
    o = run_ofm(op, method, X0, 10, refresh=0, beta_rule="pr")
    X, r = gpu_run(g, method, X0, 10, beta_rule="pr")
    assert rel(X, o.X) <= 1e-10
    assert [list(c) for c in r.codes] == [list(c) for c in o.codes]


@pytest.mark.parametrize("method", METHODS)
def test_c4_full_size_two_iterations_all_methods(method):
    """c4 at full size in the bench configuration (LPA-reordered graph): 2 iterations
    (the second with PR+ beta) of each method against the oracle on all 5M rows."""
    cfg, op, g, X0 = setup("c4", True)
    o = run_ofm(op, method, X0, 2, refresh=0)
    X, r = gpu_run(g, method, X0, 2)
    assert r.report["iters"] == 2
    assert [list(c) for c in r.codes] == [list(c) for c in o.codes]
    assert np.max(np.abs(r.alphas - np.array(o.alphas))) <= 1e-12 * np.max(np.abs(o.alphas))
    assert rel(X, o.X) <= 1e-12
    assert np.allclose(r.history[:, :2], o.history[:2, :2], rtol=1e-11, atol=0)


def test_c4_full_size_fp32():
    """fp32 storage (fp64 Grams / k x k) at c4 vs the precision-matched oracle."""
    cfg, op, g, X0 = setup("c4", True)
    X0r = X0.astype(np.float32).astype(np.float64)
    o = run_ofm(op, "ofm_f2", X0r, 5, refresh=0, precision="f32")
    X, r = gpu_run(g, "ofm_f2", X0r, 5, dtype="f32")
    assert r.report["iters"] == 5
    assert rel(X, o.X) <= 1e-4


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_p3_c2_subspace_vs_eigsh_and_oracle(method):
    cfg, op, g, X0 = setup("c2", False)
    k = cfg.k
    w, U = bottom_eigs(op, k + 2)
    assert w[k] - w[k - 1] > 0.05                        # span U_32 is well defined
    X, r = gpu_run(g, method, X0, cfg.iters)
    o = run_ofm(op, method, X0, cfg.iters, refresh=0)
    assert sines(X, U[:, :k]).max() <= 1e-6
    assert sines(o.X, U[:, :k]).max() <= 1e-6
    assert sines(X, o.X).max() <= 1e-6
    assert abs(r.history[-1, 0] - o.history[-1, 0]) <= 1e-10 * abs(o.history[-1, 0])


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_p3_c3_features_enter_cluster_band(method):
    """c3 itself: k = 64 < 71 planted blocks puts lambda_64, lambda_65 2e-4 apart
    inside the 71-eigenvalue band, so neither span U_64 nor the band is reached to
    1e-6 in a feasible run (measured, profiles/r02/c3_band.jsonl: max sine to span
    U_71 1.2e-3 at 500 iterations, 4e-5 at 4000, 3e-5 at 8000; to U_64 still O(1)).
    Asserted: the OFM objective never increases, the features approach the
    band (sines at 2000 iterations below those at 500, and below 1e-3), and their
    Ritz values lie inside [lambda_1, lambda_71]."""
    cfg, op, g, X0 = setup("c3", True)
    w, U = bottom_eigs(op, 73)
    band = 71                                            # planted blocks of c3
    assert w[band] - w[band - 1] > 0.1                   # the band is separated ...
    assert w[cfg.k] - w[cfg.k - 1] < 1e-3                # ... U_64 inside it is not
    X5, r5 = gpu_run(g, method, X0, 500)
    obj = r5.history[:, 0]
    assert np.all(np.diff(obj) <= 1e-12 * np.abs(obj[:-1]))
    X20, _ = gpu_run(g, method, X0, 2000)
    s5, s20 = sines(X5, U[:, :band]).max(), sines(X20, U[:, :band]).max()
    assert s20 < s5 and s20 <= 1e-3, (s5, s20)
    q, _ = np.linalg.qr(X20)
    Sn = sp.diags(op.s) @ op.S @ sp.diags(op.s)
    theta = np.linalg.eigvalsh(q.T @ (-q - Sn @ q))
    assert theta.min() >= w[0] - 1e-10 and theta.max() <= w[band - 1] + 1e-6


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_p3_c3_shape_separated_subspace(method):
    """The c3 shape (N = 200k, avg degree 16, 5:1, Dirichlet(5), k = 64) with 64
    planted blocks, so lambda_64 / lambda_65 are separated: OFM features reach span
    U_64 (scipy eigsh) to sines <= 1e-6 (SURVEY 8(c).4 large-N subspace pin)."""
    from synth import dcsbm_graph
    n, k = 200_000, 64
    s, d, _ = dcsbm_graph(n, 64, 1_600_000, 5.0, 321, 5.0)
    op = build_operator(n, s, d)
    w, U = bottom_eigs(op, k + 2)
    gap = w[k] - w[k - 1]
    assert gap > 0.05, gap
    g = ofsc.Graph(n, s, d, reorder=True)
    X0 = x0_block(n, k, 322)
    X, r = gpu_run(g, method, X0, 2000, tol=1e-11, check_every=50)
    sn = sines(X, U[:, :k]).max()
    assert sn <= 1e-6, (sn, r.report["iters"], r.report["grad_norm"] / r.report["grad_norm0"])
    g.close()


def test_c5_full_size_streaming_protocol():
    """c5 at full size (N = 1M, 48 blocks, 8M edges, k = 48) in the streaming launch
    configuration of tools/stream_c5.py: snapshot 1 = the first of 10
    edge-sampled parts, snapshot 2 appended in place (ofsc_graph_append) and equal,
    bit for bit, to the CSR built from the cumulative edges; on each snapshot the
    paper's 2 iterations per stage, the second snapshot warm-started from
    the first one's features, match the oracle on all rows (1e-12, same codes)."""
    from synth import stream_parts
    cfg = CONFIGS["c5"]
    s, d, _ = config_graph(cfg)
    parts = stream_parts(s, d, 10, cfg.seed_graph + 1000)
    g = ofsc.Graph(cfg.n, *parts[0])
    X = x0_block(cfg.n, cfg.k, cfg.seed_x0)
    for snap in (1, 2):
        if snap == 2:
            g.append(*parts[1])
            cs = np.concatenate([parts[0][0], parts[1][0]])
            cd = np.concatenate([parts[0][1], parts[1][1]])
            ref = ofsc.Graph(cfg.n, cs, cd)
            a, b = g.copy_csr(), ref.copy_csr()
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
            assert g.info["fro2_A"] == ref.info["fro2_A"]
            ref.close()
        else:
            cs, cd = parts[0]
        op = build_operator(cfg.n, cs, cd)
        o = run_ofm(op, "ofm_f1", X, 2, refresh=0)
        Xg, r = gpu_run(g, "ofm_f1", X, 2)
        assert [list(c) for c in r.codes] == [list(c) for c in o.codes]
        assert rel(Xg, o.X) <= 1e-12
        X = Xg                                            # warm start
    g.close()


@pytest.mark.parametrize("method", ["ofm_f1", "triofm_f2"])
def test_p2_c3_fp32(method):
    """fp32 storage at c3 (N = 200k, k = 64): 10 iterations vs the precision-matched
    oracle (P2 fp32 tolerance 1e-4)."""
    cfg, op, g, X0 = setup("c3", True)
    X0r = X0.astype(np.float32).astype(np.float64)
    o = run_ofm(op, method, X0r, 10, refresh=0, precision="f32")
    X, r = gpu_run(g, method, X0r, 10, dtype="f32")
    assert r.report["iters"] == 10
    assert rel(X, o.X) <= 1e-4

"""Oracle Algorithm 2 pins: monotone objective, theorem limits, subspaces."""
import numpy as np
import pytest

from oracle import build_operator, run_ofm, dense_A, jacobi_eigh, METHODS
from synth import CONFIGS, config_graph, x0_block
from tests import graphs as G


def sines(A, B):
    """Principal-angle sines between span(A) and span(B)."""
    qa, _ = np.linalg.qr(A)
    qb, _ = np.linalg.qr(B)
    c = np.clip(np.linalg.svd(qa.T @ qb, compute_uv=False), 0, 1)
    return np.sqrt(1 - c ** 2)


@pytest.fixture(scope="module")
def bridged():
    pairs, n = G.bridged_cliques([5, 7, 9, 12], bridges=3)
    s, d = G.edges(pairs)
    op = build_operator(n, s, d)
    w, U = jacobi_eigh(dense_A(op))
    return op, w, U


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["c1"]
    s, d, lab = config_graph(cfg)
    op = build_operator(cfg.n, s, d)
    w, U = np.linalg.eigh(dense_A(op))
    return op, w, U, x0_block(cfg.n, cfg.k, cfg.seed_x0)


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_ofm_objective_monotone(c1, method):
    op, w, U, X0 = c1
    r = run_ofm(op, method, X0, 60)
    obj = r.history[:r.iters, 0]
    assert np.all(np.diff(obj) <= 1e-10 * np.abs(obj[:-1]) + 1e-14)


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_ofm_converges_to_eigen_subspace_c1(c1, method):
    op, w, U, X0 = c1
    k = X0.shape[1]
    r = run_ofm(op, method, X0, 200)
    assert not r.diverged
    assert sines(r.X, U[:, :k]).max() <= 1e-6
    XtX = r.X.T @ r.X
    if method == "ofm_f1":     # Theorem 1: X = U_k sqrt(-Lam_k) Q  -> eig(X^T X) = -lam_1..k
        assert np.allclose(np.sort(np.linalg.eigvalsh(XtX)), np.sort(-w[:k]), atol=1e-8)
    else:                      # Theorem 3: X = U_k Q -> X^T X = I
        assert np.allclose(XtX, np.eye(k), atol=1e-8)


def test_triofm_ordered_fixed_points(bridged):
    """Theorems 2 and 4 on a well-separated spectrum: columns -> +-sqrt(-lam_i) u_i / +-u_i in order."""
    op, w, U = bridged
    k = 4
    X0 = x0_block(op.n, k, 7)
    r1 = run_ofm(op, "triofm_f1", X0, 3000, beta_rule="pr")
    d1 = np.diag(r1.X.T @ r1.X)
    assert np.allclose(d1, -w[:k], atol=1e-8)
    cos1 = np.abs(np.sum(r1.X * U[:, :k], 0)) / np.linalg.norm(r1.X, axis=0)
    assert np.allclose(cos1, 1.0, atol=1e-8)
    r2 = run_ofm(op, "triofm_f2", X0, 3000)
    assert np.allclose(r2.X.T @ r2.X, np.eye(k), atol=1e-8)
    cos2 = np.abs(np.sum(r2.X * U[:, :k], 0))
    assert np.allclose(cos2, 1.0, atol=1e-8)


def test_paper_schedule_equals_recurrence_short_horizon(c1):
    op, w, U, X0 = c1
    for m in METHODS:
        a = run_ofm(op, m, X0, 10, refresh=1)
        b = run_ofm(op, m, X0, 10, refresh=0)
        rel = np.linalg.norm(a.X - b.X) / np.linalg.norm(a.X)
        assert rel <= 1e-10, (m, rel)


def test_zero_start_is_stationary(c1):
    op, w, U, X0 = c1
    r = run_ofm(op, "ofm_f2", np.zeros_like(X0), 5)
    assert r.converged and r.iters == 0


def test_tolerance_stop(c1):
    op, w, U, X0 = c1
    r = run_ofm(op, "ofm_f1", X0, 500, tol=1e-6)
    assert r.converged and r.iters < 500
    assert r.grad_norm <= 1e-6 * 4.0 * np.linalg.norm(r.X)


def test_fixed_step_option(c1):
    op, w, U, X0 = c1
    r = run_ofm(op, "ofm_f2", X0, 50, line_search=False, alpha_fixed=0.2, beta_rule="zero")
    assert np.all(r.history[:50, 2] == 0.2)
    assert r.history[49, 0] < r.history[0, 0]


def test_fp32_mode_tracks_fp64(c1):
    op, w, U, X0 = c1
    for m in METHODS:
        a = run_ofm(op, m, X0, 10)
        b = run_ofm(op, m, X0, 10, precision="f32")
        assert np.array_equal(b.X, b.X.astype(np.float32).astype(np.float64))
        assert np.linalg.norm(a.X - b.X) / np.linalg.norm(a.X) < 1e-2


def test_row_sample_covers_the_iteration():
    """oracle/sample.py (bounded CPU timing): the row blocks partition the rows and
    the block direction / update equal the full-array ones restricted to the block."""
    from oracle import build_operator, apply_A, direction
    from oracle.sample import iteration_rows
    from synth import dcsbm_graph, x0_block
    n, k = 600, 5
    s, d, _ = dcsbm_graph(n, 4, 2400, 3.0, 5, 5.0)
    op = build_operator(n, s, d)
    X = x0_block(n, k, 6)
    AX = apply_A(op, X)
    M, W = X.T @ X, X.T @ AX
    Gp = direction("ofm_f2", X, AX, M, W)
    Vp = -Gp
    beta = np.full(k, 0.3)
    G = direction("ofm_f2", X, AX, M, W)
    V = -G + Vp * beta[None, :]
    AVp = apply_A(op, Vp)
    for r0, r1 in ((0, 200), (200, 450), (450, 600)):
        alpha, Xn, AXn = iteration_rows(op, "ofm_f2", X, AX, Gp, Vp, M, W, r0, r1, beta=beta)
        assert np.allclose(Xn, X[r0:r1] + V[r0:r1] * alpha[None, :], rtol=0, atol=1e-15)
        assert np.allclose(AXn, AX[r0:r1] + AVp[r0:r1] * alpha[None, :], rtol=0, atol=1e-14)

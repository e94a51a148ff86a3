"""Oracle direction / objective / cubic pins."""
import numpy as np
import pytest

from oracle import (build_operator, apply_A, dense_A, fro2_A, direction, objective,
                    grams, cubic_coefficients, METHODS, jacobi_eigh)
from tests import graphs as G


def small(n=30, m=90, seed=0):
    s, d = G.random_graph(n, m, seed)
    op = build_operator(n, s, d)
    return op, dense_A(op)


def f1_dense(A, X):
    return np.sum((A + X @ X.T) ** 2)


def f2_dense(A, X):
    k = X.shape[1]
    return np.trace((2 * np.eye(k) - X.T @ X) @ X.T @ A @ X)


def g_of(method, op, X):
    AX = apply_A(op, X)
    return direction(method, X, AX, X.T @ X, X.T @ AX)


@pytest.mark.parametrize("method,f", [("ofm_f1", f1_dense), ("ofm_f2", f2_dense)])
def test_gradient_matches_finite_differences(method, f):
    op, A = small()
    rng = np.random.default_rng(1)
    X = rng.standard_normal((30, 3)) * 0.3
    G_ = g_of(method, op, X)
    h = 1e-6
    fd = np.zeros_like(X)
    for i in range(30):
        for j in range(3):
            E = np.zeros_like(X)
            E[i, j] = h
            fd[i, j] = (f(A, X + E) - f(A, X - E)) / (2 * h)
    assert np.max(np.abs(fd - G_)) <= 1e-6 * np.max(np.abs(G_))


def test_k1_reductions():
    op, A = small(seed=2)
    X = np.random.default_rng(2).standard_normal((30, 1))
    assert np.allclose(g_of("triofm_f1", op, X), g_of("ofm_f1", op, X) / 4, rtol=1e-14, atol=1e-15)
    assert np.allclose(g_of("triofm_f2", op, X), g_of("ofm_f2", op, X) / 2, rtol=1e-14, atol=1e-15)


def test_objective_from_grams_equals_dense_definition():
    op, A = small(seed=3)
    X = np.random.default_rng(3).standard_normal((30, 4))
    AX = apply_A(op, X)
    M, W = X.T @ X, X.T @ AX
    assert abs(objective("ofm_f1", M, W, fro2_A(op)) - f1_dense(A, X)) <= 1e-12 * f1_dense(A, X)
    assert abs(objective("ofm_f2", M, W, 0.0) - f2_dense(A, X)) <= 1e-12 * abs(f2_dense(A, X))


def eigpairs(op, k):
    w, U = jacobi_eigh(dense_A(op))
    return w, U, w[:k], U[:, :k]


def test_theorem_fixed_points_and_minima():
    pairs, n = G.bridged_cliques([5, 7, 9, 12], bridges=3)
    s, d = G.edges(pairs)
    op = build_operator(n, s, d)
    k = 4
    w, U, lam, Uk = eigpairs(op, k)
    fro = np.sqrt(fro2_A(op))
    Q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((k, k)))
    D = np.diag([1.0, -1.0, 1.0, -1.0])
    Xf1 = Uk @ np.diag(np.sqrt(-lam))
    # Theorem 1: U_k sqrt(-Lam_k) Q stationary; Theorem 2: U_k sqrt(-Lam_k) D
    assert np.linalg.norm(g_of("ofm_f1", op, Xf1 @ Q)) <= 1e-10 * fro
    assert np.linalg.norm(g_of("triofm_f1", op, Xf1 @ D)) <= 1e-10 * fro
    # Theorem 3: U_k Q; Theorem 4: U_k D
    assert np.linalg.norm(g_of("ofm_f2", op, Uk @ Q)) <= 1e-10 * fro
    assert np.linalg.norm(g_of("triofm_f2", op, Uk @ D)) <= 1e-10 * fro
    # P:199 grad f1(U_k) != 0 ; P:243 grad f2(U_k) = 0
    assert np.linalg.norm(g_of("ofm_f1", op, Uk)) > 1e-3
    # closed-form minima: f1* = sum_{i>k} lam_i^2, f2* = sum_{i<=k} lam_i
    A = dense_A(op)
    assert abs(f1_dense(A, Xf1 @ Q) - np.sum(w[k:] ** 2)) <= 1e-10 * np.sum(w ** 2)
    assert abs(f2_dense(A, Uk @ Q) - np.sum(lam)) <= 1e-12 * abs(np.sum(lam))
    # triangular direction is NOT stationary at a rotated point (ordering matters)
    assert np.linalg.norm(g_of("triofm_f1", op, Xf1 @ Q)) > 1e-4


def exact_cubic_fit(method, op, X, V):
    """Coefficients of tr(V^T grad f(X + aV)) (OFM; /4 for f1) or diag(V^T g(X + aV))
    (Tri) from 4 direct evaluations -- an exact fit since the expression is cubic in a."""
    alphas = np.array([-1.0, 0.0, 1.0, 2.0])
    vals = []
    for a in alphas:
        Ga = g_of(method, op, X + a * V)
        if method.startswith("tri"):
            vals.append(np.einsum("ij,ij->j", V, Ga))
        else:
            vals.append(np.array([np.sum(V * Ga) / (4.0 if method == "ofm_f1" else 1.0)]))
    vals = np.array(vals)                              # [4, ncub]
    Vm = np.vander(alphas, 4)                          # columns a^3, a^2, a, 1
    return np.linalg.solve(Vm, vals)                   # [4, ncub] rows c3..c0


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_cubic_coefficients_equal_exact_fit(method, seed):
    op, A = small(60, 200, seed)
    rng = np.random.default_rng(seed)
    k = 4
    X = rng.standard_normal((60, k)) * 0.3
    V = rng.standard_normal((60, k)) * 0.2
    AX, AV = apply_A(op, X), apply_A(op, V)
    Q, P, T, Rp = grams(V, X, AV)
    c = np.array([np.atleast_1d(x) for x in
                  cubic_coefficients(method, Q, P, T, Rp, X.T @ X, X.T @ AX)])
    fit = exact_cubic_fit(method, op, X, V)
    scale = np.max(np.abs(fit))
    assert np.max(np.abs(c - fit)) <= 1e-11 * scale


def test_cubic_x_zero_special_cases():
    op, A = small(seed=4)
    V = np.random.default_rng(4).standard_normal((30, 3))
    X = np.zeros_like(V)
    AV = apply_A(op, V)
    Q, P, T, Rp = grams(V, X, AV)
    c3, c2, c1, c0 = cubic_coefficients("ofm_f1", Q, P, T, Rp, X.T @ X, X.T @ apply_A(op, X))
    assert c2 == 0.0 and c0 == 0.0
    assert np.isclose(c3, np.trace(Q @ Q)) and np.isclose(c1, np.trace(T))
    c3, c2, c1, c0 = cubic_coefficients("ofm_f2", Q, P, T, Rp, X.T @ X, X.T @ apply_A(op, X))
    assert c2 == 0.0 and c0 == 0.0 and np.isclose(c3, -4 * np.trace(Q @ T)) and np.isclose(c1, 4 * np.trace(T))


def test_k1_tri_cubic_equals_ofm_cubic():
    op, A = small(seed=5)
    rng = np.random.default_rng(5)
    X, V = rng.standard_normal((30, 1)), rng.standard_normal((30, 1))
    AX, AV = apply_A(op, X), apply_A(op, V)
    Q, P, T, Rp = grams(V, X, AV)
    M, W = X.T @ X, X.T @ AX
    t1 = np.array(cubic_coefficients("triofm_f1", Q, P, T, Rp, M, W)).ravel()
    o1 = np.array(cubic_coefficients("ofm_f1", Q, P, T, Rp, M, W))
    assert np.allclose(t1, o1, rtol=1e-13)
    t2 = np.array(cubic_coefficients("triofm_f2", Q, P, T, Rp, M, W)).ravel()
    o2 = np.array(cubic_coefficients("ofm_f2", Q, P, T, Rp, M, W))
    assert np.allclose(t2, o2 / 2, rtol=1e-13)


def test_psi_equals_objective_difference():
    """OFM: psi(a) = (f(X+aV) - f(X))/4 (f1) and f2(X+aV) - f2(X) (f2)."""
    from oracle import psi
    op, A = small(seed=6)
    rng = np.random.default_rng(6)
    X, V = rng.standard_normal((30, 3)) * 0.3, rng.standard_normal((30, 3)) * 0.3
    AX, AV = apply_A(op, X), apply_A(op, V)
    Q, P, T, Rp = grams(V, X, AV)
    for method, f, sc in (("ofm_f1", f1_dense, 4.0), ("ofm_f2", f2_dense, 1.0)):
        c = cubic_coefficients(method, Q, P, T, Rp, X.T @ X, X.T @ AX)
        for a in (-0.7, 0.3, 1.1):
            lhs = psi(*c, a)
            rhs = (f(A, X + a * V) - f(A, X)) / sc
            assert abs(lhs - rhs) <= 1e-11 * (abs(rhs) + 1.0)

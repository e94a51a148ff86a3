"""Pins of the oracle's orthogonalisation + Rayleigh-Ritz step and relerr
(SURVEY 8(f) NEXT-1).  Each pin is fixed by mathematics the
oracle does not use itself: LAPACK eigh of the dense operator, the
Courant-Fischer bounds, the dense B = L + 2I matrix of P:589."""
import numpy as np
import pytest

from oracle import build_operator, dense_A
from oracle.rr import rayleigh_ritz
from tests import graphs as G


def small(n=40, m=140, seed=0):
    s, d = G.random_graph(n, m, seed)
    op = build_operator(n, s, d)
    return op, dense_A(op)


@pytest.mark.parametrize("k", [1, 3, 6])
def test_exact_eigenvectors_give_eigenpairs(k):
    """X = U_k (LAPACK): Ritz values = the k smallest eigenvalues, relerr = 0."""
    op, A = small()
    lam, U = np.linalg.eigh(A)
    r = rayleigh_ritz(op, U[:, :k])
    assert np.allclose(r.theta, lam[:k], atol=1e-12, rtol=0)
    assert r.relerr <= 1e-12


def test_invariant_under_basis_change():
    """span(X G) = span(X): same Ritz values and relerr, same Ritz vectors up to sign."""
    op, A = small(seed=3)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((op.n, 5))
    Gm = rng.standard_normal((5, 5)) + 3 * np.eye(5)
    r1, r2 = rayleigh_ritz(op, X), rayleigh_ritz(op, X @ Gm)
    assert np.allclose(r1.theta, r2.theta, atol=1e-11, rtol=0)
    assert abs(r1.relerr - r2.relerr) <= 1e-10
    sg = np.sign(np.sum(r1.U * r2.U, axis=0))
    assert np.allclose(r1.U, r2.U * sg[None, :], atol=1e-9)


def test_courant_fischer_and_orthonormality():
    """Random subspace: theta_i >= lambda_i (Courant-Fischer), theta_i <= lambda_max,
    U^T U = I, U^T A U = diag(theta) against the dense operator."""
    op, A = small(n=60, m=200, seed=5)
    lam = np.linalg.eigvalsh(A)
    rng = np.random.default_rng(2)
    for k in (2, 7, 12):
        X = rng.standard_normal((op.n, k))
        r = rayleigh_ritz(op, X)
        assert np.all(r.theta >= lam[:k] - 1e-12)
        assert np.all(r.theta <= lam[-1] + 1e-12)
        assert np.allclose(r.U.T @ r.U, np.eye(k), atol=1e-12)
        assert np.allclose(r.U.T @ A @ r.U, np.diag(r.theta), atol=1e-12)


def test_full_subspace_gives_the_spectrum():
    """k = n: the Ritz values are the whole spectrum (LAPACK) and relerr = 0."""
    op, A = small(n=25, m=70, seed=8)
    rng = np.random.default_rng(3)
    r = rayleigh_ritz(op, rng.standard_normal((op.n, op.n)))
    assert np.allclose(r.theta, np.linalg.eigvalsh(A), atol=1e-12, rtol=0)
    assert r.relerr <= 1e-12


def test_relerr_is_the_paper_formula_with_dense_B():
    """P:589 with B = L + 2I built densely from S (R26): ||B U - U Lam_B|| / ||U Lam_B||."""
    op, A = small(n=50, m=160, seed=11)
    S = op.S.toarray()
    d = S.sum(axis=1)
    dih = np.where(d > 0, 1.0 / np.sqrt(np.maximum(d, 1)), 0.0)
    Lap = np.eye(op.n) - dih[:, None] * S * dih[None, :]
    B = Lap + 2.0 * np.eye(op.n)
    rng = np.random.default_rng(4)
    X = rng.standard_normal((op.n, 4))
    r = rayleigh_ritz(op, X)
    lamB = r.theta + 4.0
    ref = np.linalg.norm(B @ r.U - r.U * lamB[None, :]) / np.linalg.norm(r.U * lamB[None, :])
    assert abs(r.relerr - ref) <= 1e-13 * max(1.0, ref)
    assert r.relerr > 1e-3                       # a random subspace is far from invariant


def test_clique_union_block_indicators():
    """Union of c cliques, X = block indicators: theta = -2 (c times), relerr = 0,
    Ritz vectors span the normalised indicators."""
    pairs, n = G.clique_union([5, 7, 4])
    s, d = G.edges(pairs)
    op = build_operator(n, s, d)
    X = np.zeros((n, 3))
    X[:5, 0] = 1
    X[5:12, 1] = 1
    X[12:, 2] = 1
    r = rayleigh_ritz(op, X)
    assert np.allclose(r.theta, -2.0, atol=1e-13)
    assert r.relerr <= 1e-13
    P = r.U @ r.U.T
    Xn = X / np.linalg.norm(X, axis=0)
    assert np.allclose(P, Xn @ Xn.T, atol=1e-13)


def test_rank_deficient_subspace_raises():
    op, A = small()
    X = np.ones((op.n, 2))
    with pytest.raises(np.linalg.LinAlgError):
        rayleigh_ritz(op, X)

"""Oracle clustering pins: row normalise, Lloyd, ARI/NMI, Jacobi."""
import itertools

import numpy as np
import pytest

from oracle import (row_normalize, kmeans_lloyd, ari, nmi, jacobi_eigh, build_operator,
                    run_ofm)
from synth import x0_block
from tests import graphs as G


def test_row_normalize():
    Y = row_normalize(np.array([[3.0, 4.0], [0.0, 0.0], [1.0, 0.0]]))
    assert np.allclose(Y, [[0.6, 0.8], [0.0, 0.0], [1.0, 0.0]], atol=1e-16)


def test_ari_nmi_examples():
    assert ari([0, 0, 1, 1], [0, 1, 0, 1]) == pytest.approx(-0.5, abs=1e-12)
    assert nmi([0, 0, 1, 1], [0, 1, 0, 1]) == pytest.approx(0.0, abs=1e-12)
    assert ari([0, 0, 1, 2], [5, 5, 7, 3]) == 1.0
    assert nmi([0, 0, 1, 2], [5, 5, 7, 3]) == pytest.approx(1.0)
    assert nmi([0, 0, 1, 1], [0, 0, 0, 0]) == 0.0


@pytest.mark.parametrize("seed", range(20))
def test_ari_nmi_symmetric_and_permutation_invariant(seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 4, 30)
    b = rng.integers(0, 5, 30)
    perm = rng.permutation(5)
    assert ari(a, b) == pytest.approx(ari(b, a), abs=1e-12)
    assert ari(a, b) == pytest.approx(ari(a, perm[b]), abs=1e-12)
    assert nmi(a, b) == pytest.approx(nmi(b, a), abs=1e-12)
    assert ari(a, b) <= 1.0


def brute_best_partition(Y, K):
    best, bestl = np.inf, None
    n = Y.shape[0]
    for lab in itertools.product(range(K), repeat=n):
        lab = np.array(lab)
        if len(set(lab)) < K:
            continue
        cost = sum(np.sum((Y[lab == c] - Y[lab == c].mean(0)) ** 2) for c in range(K))
        if cost < best - 1e-12:
            best, bestl = cost, lab
    return best, bestl


@pytest.mark.parametrize("seed", range(5))
def test_kmeans_reaches_brute_force_optimum_small(seed):
    rng = np.random.default_rng(seed)
    centers = np.array([[0, 0], [5, 5], [0, 6]], float)
    Y = np.concatenate([c + 0.3 * rng.standard_normal((2 + (seed % 2), 2)) for c in centers])
    best, bl = brute_best_partition(Y, 3)
    lab, C, it, inertia = kmeans_lloyd(Y, Y[[0, 3 if seed % 2 else 2, len(Y) - 1]])
    assert inertia == pytest.approx(best, rel=1e-12)
    assert ari(lab, bl) == 1.0


def test_kmeans_k1_and_blobs_and_monotone_inertia():
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((50, 3))
    lab, C, _, _ = kmeans_lloyd(Y, Y[:1])
    assert np.all(lab == 0) and np.allclose(C[0], Y.mean(0))
    truth = np.repeat([0, 1], 40)
    Yb = np.concatenate([rng.standard_normal((40, 2)), 10 + rng.standard_normal((40, 2))])
    lab, _, _, _ = kmeans_lloyd(Yb, Yb[[0, 1]])
    assert ari(lab, truth) == 1.0
    Y = rng.standard_normal((300, 4))
    prev = np.inf
    for m in range(1, 8):
        _, _, _, inertia = kmeans_lloyd(Y, Y[:6], max_iters=m)
        assert inertia <= prev + 1e-12
        prev = inertia


def test_kmeans_tie_goes_to_lowest_index_and_empty_keeps():
    Y = np.array([[0.0], [2.0]])
    lab, C, _, _ = kmeans_lloyd(Y, np.array([[1.0], [1.0], [50.0]]), max_iters=1)
    assert list(lab) == [0, 0]
    assert C[2, 0] == 50.0 and C[1, 0] == 1.0


def test_clique_union_end_to_end_ari_one():
    pairs, n = G.clique_union([6, 8, 10])
    s, d = G.edges(pairs)
    op = build_operator(n, s, d)
    r = run_ofm(op, "ofm_f2", x0_block(n, 3, 1), 300)
    Y = row_normalize(r.X)
    truth = np.repeat([0, 1, 2], [6, 8, 10])
    lab, _, _, _ = kmeans_lloyd(Y, Y[[0, 6, 14]])
    assert ari(lab, truth) == 1.0


def test_jacobi_textbook_and_cross_check():
    w, V = jacobi_eigh(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(w, [1.0, 3.0], atol=1e-15)
    assert np.allclose(np.abs(V), np.full((2, 2), 1 / np.sqrt(2)), atol=1e-15)
    assert np.allclose(jacobi_eigh(np.diag([3.0, -1.0, 2.0]))[0], [-1.0, 2.0, 3.0])
    rng = np.random.default_rng(0)
    for n in (5, 17, 40):
        B = rng.standard_normal((n, n))
        A = B + B.T
        w, V = jacobi_eigh(A)
        assert np.allclose(w, np.linalg.eigvalsh(A), atol=1e-12 * np.abs(w).max())
        assert np.linalg.norm(V @ np.diag(w) @ V.T - A) <= 1e-10 * np.linalg.norm(A)
        assert np.allclose(V.T @ V, np.eye(n), atol=1e-12)

"""Oracle operator pins: closed-form spectra of A = L - 2I."""
import math

import numpy as np
import pytest

from oracle import build_operator, apply_A, dense_A, fro2_A
from tests import graphs as G


def op_of(pairs, n=None):
    s, d = G.edges(pairs)
    if n is None:
        n = int(max(s.max(), d.max())) + 1
    return build_operator(n, s, d)


def spec(op):
    return np.sort(np.linalg.eigvalsh(dense_A(op)))


def test_two_node_closed_form():
    op = op_of([(0, 1)])
    assert np.array_equal(dense_A(op), np.array([[-1.0, -1.0], [-1.0, -1.0]]))
    assert np.allclose(spec(op), [-2.0, 0.0], atol=1e-14)


def test_path3_spectrum():
    assert np.allclose(spec(op_of(G.path(3))), [-2.0, -1.0, 0.0], atol=1e-13)


@pytest.mark.parametrize("n", [3, 5, 8])
def test_clique_spectrum(n):
    w = spec(op_of(G.clique(n)))
    expect = np.sort([-2.0] + [-(n - 2) / (n - 1)] * (n - 1))
    assert np.allclose(w, expect, atol=1e-12)


@pytest.mark.parametrize("n", [4, 7, 12])
def test_cycle_spectrum(n):
    w = spec(op_of(G.cycle(n)))
    expect = np.sort([-1.0 - math.cos(2 * math.pi * j / n) for j in range(n)])
    assert np.allclose(w, expect, atol=1e-12)


def test_star_and_bipartite_have_zero_eigenvalue():
    w = spec(op_of(G.star(5)))
    assert np.allclose(w, np.sort([-2.0, 0.0] + [-1.0] * 4), atol=1e-12)
    w = spec(op_of(G.complete_bipartite(3, 4)))
    assert abs(w[-1]) < 1e-12 and abs(w[0] + 2.0) < 1e-12


def test_clique_union_eigenvectors_are_block_indicators():
    pairs, n = G.clique_union([4, 6, 5])
    op = op_of(pairs, n)
    w, U = np.linalg.eigh(dense_A(op))
    assert np.allclose(w[:3], -2.0, atol=1e-12) and w[3] > -2.0 + 1e-3
    ind = np.zeros((n, 3))
    ind[0:4, 0] = 1 / 2.0
    ind[4:10, 1] = 1 / math.sqrt(6)
    ind[10:15, 2] = 1 / math.sqrt(5)
    # same subspace: projector equality
    assert np.allclose(U[:, :3] @ U[:, :3].T, ind @ ind.T, atol=1e-12)


def test_sqrt_degree_vector_and_isolated_node():
    s, d = G.random_graph(40, 120, 3)
    op = build_operator(45, s, d)            # nodes 40..44 isolated
    A = dense_A(op)
    v = np.sqrt(op.deg.astype(float))
    assert np.allclose(A @ v, -2.0 * v, atol=1e-12)          # D^{1/2} 1, lambda(L) = 0
    e = np.zeros(45)
    e[44] = 1.0
    assert np.array_equal(A @ e, -e)                          # isolated: row -e_i
    assert op.s[44] == 0.0


@pytest.mark.parametrize("seed", range(10))
def test_random_spectrum_in_range_and_symmetric(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 60))
    s, d = G.random_graph(n, int(rng.integers(1, 4 * n)), seed)
    op = build_operator(n, s, d)
    A = dense_A(op)
    assert np.array_equal(A, A.T)
    w = np.linalg.eigvalsh(A)
    assert w.min() >= -2.0 - 1e-12 and w.max() <= 1e-12
    # multiplicity of -2 = number of non-trivial components
    import scipy.sparse.csgraph as csg
    ncomp, lab = csg.connected_components(op.S, directed=False)
    nontriv = sum(1 for c in range(ncomp) if op.deg[lab == c].sum() > 0)
    assert np.sum(np.abs(w + 2.0) < 1e-9) == nontriv


@pytest.mark.parametrize("seed", range(4))
def test_apply_equals_dense_definition_and_fro2(seed):
    n = 200
    s, d = G.random_graph(n, 700, 10 + seed)
    op = build_operator(n, s, d)
    # dense definition written from P:28-31 directly: adjacency from the edge list
    Sd = np.zeros((n, n))
    for a, b in zip(s, d):
        if a != b:
            Sd[a, b] = Sd[b, a] = 1.0
    deg = Sd.sum(1)
    dinv = np.where(deg > 0, 1.0 / np.sqrt(np.maximum(deg, 1)), 0.0)
    L = np.eye(n) - np.diag(dinv) @ Sd @ np.diag(dinv)
    A = L - 2.0 * np.eye(n)
    Z = np.random.default_rng(seed).standard_normal((n, 7))
    assert np.allclose(apply_A(op, Z), A @ Z, rtol=1e-14, atol=1e-14)
    assert abs(fro2_A(op) - np.sum(A * A)) <= 1e-12 * np.sum(A * A)


def test_build_canonicalises_and_counts():
    op = build_operator(4, np.array([0, 1, 1, 2, 3, 3]), np.array([1, 0, 1, 3, 2, 2]))
    assert op.n_edges == 2 and op.n_self_loops == 1 and op.n_duplicates == 3
    assert list(op.row_ptr) == [0, 1, 2, 3, 4] and list(op.col) == [1, 0, 3, 2]
    with pytest.raises(IndexError):
        build_operator(3, np.array([0]), np.array([3]))


def test_fp32_apply_close_to_fp64():
    s, d = G.random_graph(300, 2000, 7)
    op = build_operator(300, s, d)
    Z = np.random.default_rng(1).standard_normal((300, 16)).astype(np.float32).astype(np.float64)
    y32 = apply_A(op, Z, "f32")
    y64 = apply_A(op, Z)
    assert np.array_equal(y32, y32.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(y32 - y64)) < 1e-5 * np.max(np.abs(y64))

"""Oracle pins of the column-wise CG rule and the summation rule.

beta (Alg. 2 l.9): beta_i = sum_r (G - Gp)_ri G_ri / sum_r Gp_ri^2, PR+
clamp (R5), 0 when the denominator is 0 (SURVEY 8(c).4 "beta" row,
S:332-334).  The integer-valued cases below make every quantity exact, so the
pins are equalities.  The wiring of run_ofm (V_1 = -G_1 + beta_1 V_0) is pinned
against directions recomputed from the dense operator.

Summation rule (R29): 1024-row blocks, block
sums combined pairwise in block order; pinned against exactly rounded sums
(math.fsum) and against the order it states.
"""
import math

import numpy as np
import pytest

from oracle import (beta_pr, build_operator, colsum, dense_A, direction, gram, pairwise_sum,
                    run_ofm)
from synth import dcsbm_graph, x0_block


def test_beta_zero_when_gradient_repeats():
    """G = Gp: (G - Gp) . G = 0, so beta = 0 under PR and PR+."""
    rng = np.random.default_rng(0)
    G = rng.standard_normal((50, 4))
    gg = np.sum(G * G, axis=0)
    for rule in ("pr", "pr+"):
        assert np.array_equal(beta_pr(G, G.copy(), gg, rule), np.zeros(4))


def test_beta_orthogonal_columns_is_ratio_of_norms():
    """G_i orthogonal to Gp_i: beta_i = ||G_i||^2 / ||Gp_i||^2."""
    G = np.array([[1.0, 0.0], [2.0, 3.0], [0.0, 0.0], [0.0, 4.0]])
    Gp = np.array([[0.0, 1.0], [0.0, 0.0], [3.0, 2.0], [4.0, 0.0]])
    gg_prev = np.sum(Gp * Gp, axis=0)                   # 25, 5
    want = np.array([5.0 / 25.0, 25.0 / 5.0])
    for rule in ("pr", "pr+"):
        assert np.array_equal(beta_pr(G, Gp, gg_prev, rule), want)


def test_beta_pr_plus_clamps_negative():
    """G = Gp / 2: (G - Gp) . G = -||Gp||^2 / 4 -> PR gives -1/4, PR+ gives 0."""
    Gp = np.array([[2.0, 4.0], [4.0, 0.0], [0.0, 2.0]])
    G = Gp / 2.0
    gg_prev = np.sum(Gp * Gp, axis=0)
    assert np.array_equal(beta_pr(G, Gp, gg_prev, "pr"), np.array([-0.25, -0.25]))
    assert np.array_equal(beta_pr(G, Gp, gg_prev, "pr+"), np.array([0.0, 0.0]))


def test_beta_zero_denominator_and_zero_rule():
    """||Gp_i|| = 0 -> beta_i = 0 (no division); rule "zero" -> steepest descent."""
    G = np.array([[1.0, 1.0], [1.0, 2.0]])
    Gp = np.array([[0.0, 1.0], [0.0, 0.0]])
    gg_prev = np.sum(Gp * Gp, axis=0)
    b = beta_pr(G, Gp, gg_prev, "pr")
    assert b[0] == 0.0 and b[1] == (0.0 * 1.0 + 2.0 * 2.0) / 1.0
    assert np.array_equal(beta_pr(G, Gp, gg_prev, "zero"), np.zeros(2))
    with pytest.raises(ValueError):
        beta_pr(G, Gp, gg_prev, "fr")


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
@pytest.mark.parametrize("rule", ["pr", "pr+"])
def test_run_ofm_second_direction_uses_printed_beta(method, rule):
    """run_ofm's V_1 equals -G_1 + beta_1 V_0 with beta_1 from the printed formula,
    where G_0, G_1 are recomputed from the DENSE operator at X_0 and X_1 (not from
    the oracle's recurrences) and V_1 is read back from X_2 = X_1 + alpha_1 V_1."""
    n, k = 200, 3
    s, d, _ = dcsbm_graph(n, 3, 900, 3.0, 11, 5.0)
    op = build_operator(n, s, d)
    A = dense_A(op)
    X0 = x0_block(n, k, 12)

    def g_dense(X):
        AX = A @ X
        return direction(method, X, AX, X.T @ X, X.T @ AX)

    r1 = run_ofm(op, method, X0, 1, beta_rule=rule, refresh=0)
    r2 = run_ofm(op, method, X0, 2, beta_rule=rule, refresh=0)
    G0, G1 = g_dense(X0), g_dense(r1.X)
    num = np.sum((G1 - G0) * G1, axis=0)
    beta = num / np.sum(G0 * G0, axis=0)
    if rule == "pr+":
        beta = np.maximum(beta, 0.0)
    assert np.allclose(r2.betas[1], beta, rtol=1e-9, atol=1e-12)
    assert np.array_equal(r2.betas[0], np.zeros(k))
    a1 = r2.alphas[1][0]
    V1 = (r2.X - r1.X) / a1
    want = -G1 + (-G0) * beta[None, :]                 # V_0 = -G_0 (Alg. 2 l.4)
    assert np.linalg.norm(V1 - want) <= 1e-7 * np.linalg.norm(want)


def test_colsum_and_gram_match_exact_sums():
    """Blocked pairwise sums agree with exactly rounded sums (fsum) to a few ulps,
    including a ragged tail block (n = 5000 = 4 x 1024 + 904)."""
    rng = np.random.default_rng(3)
    n = 5000
    A = rng.standard_normal((n, 3)) * np.exp(rng.uniform(-3, 3, (n, 1)))
    B = rng.standard_normal((n, 2))
    cs = colsum(A)
    for j in range(3):
        ex = math.fsum(A[:, j])
        assert abs(cs[j] - ex) <= 1e-14 * math.fsum(np.abs(A[:, j]))
    gr = gram(A, B)
    for i in range(3):
        for j in range(2):
            prod = A[:, i] * B[:, j]                       # products rounded once, as in the rule
            ex = math.fsum(prod)
            assert abs(gr[i, j] - ex) <= 1e-14 * math.fsum(np.abs(prod))
    assert np.array_equal(colsum(np.zeros((0, 2))), np.zeros(2))


def test_pairwise_sum_order():
    """((p0 + p1) + (p2 + p3)) + p4: values chosen so that any other order rounds differently."""
    p = np.array([1.0, 2.0 ** -53, 2.0 ** -53, 2.0 ** -53, 2.0 ** -53])
    # p0 + p1 = 1 (tie to even), p2 + p3 = 2^-52, 1 + 2^-52 = 1 + ulp,
    # (1 + ulp) + 2^-53 is a tie -> the even neighbour 1 + 2 ulp
    assert pairwise_sum(p) == 1.0 + 2.0 ** -51
    seq = 0.0
    for x in p:
        seq += x
    assert seq == 1.0                                      # the sequential order differs
    q = np.arange(7, dtype=np.float64)[:, None] * np.ones((7, 2))
    assert np.array_equal(pairwise_sum(q), np.full(2, 21.0))

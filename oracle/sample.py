"""Oracle: one iteration of Algorithm 2 restricted to a block of rows, for
BOUNDED CPU timing only (TEST INFRASTRUCTURE ONLY: used by bench.py's
cpu_baseline and --impl reference legs, never by the product path).

A full oracle iteration at c4 (N = 5M) takes ~20 s on the host; the benchmark
contract asks for a bounded sample of the workload.  Every N-length step of an
iteration (the SpMM A V, the Grams, the direction, the update) is a sum or map
over rows, so its cost is the sum of per-row costs: this module runs exactly
the arithmetic of `methods.run_ofm`'s loop body (same functions: `direction`,
`grams`, `cubic_coefficients`, `select_step`; the SpMM is `apply_A`'s formula
-Z - s (S (s Z)) on the block's rows of S) on rows [r0, r1) with the k x k
line search done once, and the caller scales the time by N / (r1 - r0).
Two deviations, both cost-neutral: a block cannot see the new direction of the
other rows, so its SpMM gathers the previous direction Vp (same sparsity,
same flops and bytes as A V), and its beta numerator sums the block's rows
only (the denominator ||Gp_i||^2 is the previous iteration's full column sum,
`gg_prev`, computed untimed by the caller, as Alg. 2 l.9 and
`methods.beta_pr` divide).  The numbers it produces are not used for parity;
the timed arithmetic is the oracle's own, untuned.
"""
from __future__ import annotations

import numpy as np

from .cubic import select_step
from .methods import beta_pr, colsum, cubic_coefficients, direction, grams


def iteration_rows(op, method, X, AX, Gp, Vp, M, W, r0, r1, beta=None, S_rows=None, sVp=None,
                   gg_prev=None, beta_rule="pr+"):
    """One Algorithm-2 iteration on rows [r0, r1).  X, AX, Gp, Vp are
    full n x k arrays (V is gathered through S at all rows); returns alpha.
    gg_prev = sum_r Gp_ri^2 over ALL rows (the PR denominator); when None
    it is the block's own column sums of Gp.
    S_rows = op.S[r0:r1] and sVp = s * Vp (all rows) may be passed precomputed:
    the block's share of s * Vp is then recomputed inside (its per-block cost)."""
    k = X.shape[1]
    rows = slice(r0, r1)
    G = direction(method, X[rows], AX[rows], M, W)                  # Alg. 2 l.8
    gg = colsum(G * G)                                              # ||G_i||^2 (next gg_prev)
    if beta is None:                                                # Alg. 2 l.9
        if gg_prev is None:
            gg_prev = colsum(Gp[rows] * Gp[rows])
        beta = beta_pr(G, Gp[rows], gg_prev, beta_rule)
    V = -G + Vp[rows] * beta[None, :]                               # Alg. 2 l.10
    s = op.s[:, None]
    if S_rows is None:
        S_rows = op.S[r0:r1]
    if sVp is None:
        sVp = s * Vp
    else:
        sVp[rows] = s[rows] * Vp[rows]                              # this block's share of s * V
    AVb = -Vp[rows] - s[rows] * (S_rows @ sVp)                      # A V on the block's rows
    Q, P, T, Rp = grams(V, X[rows], AVb)
    c3, c2, c1, c0 = cubic_coefficients(method, Q, P, T, Rp, M, W)  # Alg. 2 l.11
    if method.startswith("tri"):
        alpha = np.array([select_step(float(c3[i]), float(c2[i]), float(c1[i]), float(c0[i]))[0]
                          for i in range(k)])
    else:
        alpha = np.full(k, select_step(float(c3), float(c2), float(c1), float(c0))[0])
    Xn = X[rows] + V * alpha[None, :]                               # Alg. 2 l.12
    AXn = AX[rows] + AVb * alpha[None, :]
    return alpha, Xn, AXn

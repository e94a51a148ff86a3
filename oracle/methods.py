"""Oracle: the four orthogonalization-free methods, Algorithm 2 (TEST INFRASTRUCTURE ONLY).

Directions (triu keeps the diagonal, R15):
  OFM-f1     grad f1 = 4AX + 4X X^T X                        eq:gradientf1
  TriOFM-f1  g1      = AX + X triu(X^T X)                    eq:gradientg1
  OFM-f2     grad f2 = 4AX - 2X X^T A X - 2AX X^T X          eq:gradientf2
  TriOFM-f2  g2      = 2AX - AX triu(X^T X) - X triu(X^T AX) eq:gradientg2
Objectives: f1 = ||A + XX^T||_F^2, f2 = tr((2I - X^T X) X^T A X).
Line-search cubics: eq:f1-derivative, eq:alphai-f1,
eq:f2-derivative, eq:alphai-f2, in terms of the Grams
Q = V^T V, P = V^T X, T = V^T A V, R' = X^T A V, R = R'^T (= V^T A X, "the
transpose of X^T A V"), M = X^T X, W = X^T A X.
Algorithm 2: G = g(X); beta = sumeachcol((G - Gp).G) / sumeachcol(Gp.Gp)
(column-wise Polak-Ribiere, with PR+ clamp by default, R5); V = -G + beta.Vp;
exact line search; X_i += alpha_i V_i.

Summation rule for every reduction over the N rows (Grams, column dots; SURVEY
8(c).2 step 2, R29): sums over fixed 1024-row blocks, then the block
sums combined pairwise in block order, so the oracle's own rounding stays at
~u (1024 + log2(N/1024)) at N = 5M instead of growing with N.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cubic import select_step, BRANCH
from .operator import Operator, apply_A, fro2_A

METHODS = ("ofm_f1", "triofm_f1", "ofm_f2", "triofm_f2")
_C_M = {"ofm_f1": 4.0, "triofm_f1": 1.0, "ofm_f2": 2.0, "triofm_f2": 1.0}


def stop_constant(method: str) -> float:
    """c_m of the scale-free stopping rule ||G||_F <= tol c_m ||X||_F (R14)."""
    return _C_M[method]


def direction(method, X, AX, M, W):
    """G = g_m(X) from X, AX, M = X^T X, W = X^T A X."""
    if method == "ofm_f1":
        return 4.0 * AX + 4.0 * (X @ M)
    if method == "triofm_f1":
        return AX + X @ np.triu(M)
    if method == "ofm_f2":
        return 4.0 * AX - 2.0 * (X @ W) - 2.0 * (AX @ M)
    if method == "triofm_f2":
        return 2.0 * AX - AX @ np.triu(M) - X @ np.triu(W)
    raise ValueError(method)


def objective(method, M, W, fro2):
    """f1 = ||A||_F^2 + 2 tr(X^T A X) + ||X^T X||_F^2 ;  f2 = 2 tr W - tr(M W)."""
    if method in ("ofm_f1", "triofm_f1"):
        return fro2 + 2.0 * np.trace(W) + np.sum(M * M)
    return 2.0 * np.trace(W) - np.sum(M * W.T)


BLOCK_ROWS = 1024


def pairwise_sum(parts):
    """Sum of parts[0], parts[1], ... combined pairwise in order: ((p0+p1)+(p2+p3))+..."""
    parts = np.asarray(parts)
    if parts.shape[0] == 0:
        return np.zeros(parts.shape[1:])
    while parts.shape[0] > 1:
        m = parts.shape[0] // 2
        nxt = parts[0:2 * m:2] + parts[1:2 * m:2]
        parts = np.concatenate([nxt, parts[2 * m:]]) if parts.shape[0] % 2 else nxt
    return parts[0]


def _row_blocks(Z):
    """Z's rows as full 1024-row blocks (a view) plus the ragged tail block (or None)."""
    n = Z.shape[0]
    nb = n // BLOCK_ROWS
    full = Z[:nb * BLOCK_ROWS].reshape((nb, BLOCK_ROWS) + Z.shape[1:])
    tail = Z[nb * BLOCK_ROWS:] if n % BLOCK_ROWS else None
    return full, tail


def colsum(Z):
    """sum_r Z[r, :] by the summation rule (1024-row blocks, pairwise over blocks)."""
    full, tail = _row_blocks(np.asarray(Z, dtype=np.float64))
    parts = full.sum(axis=1)
    if tail is not None:
        parts = np.concatenate([parts, tail.sum(axis=0)[None]])
    return pairwise_sum(parts)


def gram(A, B):
    """A^T B = sum_r A[r]^T B[r] by the summation rule (1024-row blocks, pairwise)."""
    fa, ta = _row_blocks(np.asarray(A, dtype=np.float64))
    fb, tb = _row_blocks(np.asarray(B, dtype=np.float64))
    parts = np.matmul(fa.transpose(0, 2, 1), fb)
    if ta is not None:
        parts = np.concatenate([parts, (ta.T @ tb)[None]])
    return pairwise_sum(parts)


def grams(V, X, AV):
    """Q = V^T V, P = V^T X, T = V^T (AV), R' = X^T (AV)."""
    return gram(V, V), gram(V, X), gram(V, AV), gram(X, AV)


def beta_pr(G, Gp, gg_prev, rule="pr+"):
    """Column-wise Polak-Ribiere (Alg. 2 l.9):
    beta_i = sum_r (G - Gp)_ri G_ri / sum_r Gp_ri^2, 0 where the denominator is 0;
    rule "pr+" clamps at 0 (R5), "pr" is the printed formula, "zero" gives 0.
    gg_prev = sum_r Gp_ri^2 (column sums kept from the previous iteration)."""
    k = G.shape[1]
    if rule == "zero":
        return np.zeros(k)
    num = colsum((G - Gp) * G)
    den = np.asarray(gg_prev, dtype=np.float64)
    beta = np.where(den > 0.0, num / np.where(den > 0.0, den, 1.0), 0.0)
    if rule == "pr+":
        beta = np.maximum(beta, 0.0)
    elif rule != "pr":
        raise ValueError(rule)
    return beta


def _d(A, B):
    """diag(A B)_i = sum_j A_ij B_ji."""
    return np.einsum("ij,ji->i", A, B)


def cubic_coefficients(method, Q, P, T, Rp, M, W):
    """(c3, c2, c1, c0): scalars for OFM, length-k arrays for TriOFM."""
    R = Rp.T
    U = np.triu
    tr = np.trace
    if method == "ofm_f1":          # eq:f1-derivative, printed coefficients (= phi'/4, R1)
        return (tr(Q @ Q), 3.0 * tr(Q @ P.T),
                tr(T) + tr(P @ P) + tr(P @ P.T) + tr(Q @ M),
                tr(R) + tr(P @ M))
    if method == "ofm_f2":          # eq:f2-derivative
        return (-4.0 * tr(Q @ T),
                -6.0 * (tr(P @ T) + tr(Q @ R)),
                2.0 * (2.0 * tr(T) - 2.0 * tr(P @ Rp) - 2.0 * tr(P @ R) - tr(Q @ W) - tr(M @ T)),
                2.0 * (2.0 * tr(R) - tr(P @ W) - tr(M @ R)))
    if method == "triofm_f1":       # eq:alphai-f1, i-th diagonal entries (R2)
        return (_d(Q, U(Q)),
                _d(Q, U(P.T)) + _d(Q, U(P)) + _d(P, U(Q)),
                np.diag(T) + _d(P, U(P)) + _d(P, U(P.T)) + _d(Q, U(M)),
                np.diag(R) + _d(P, U(M)))
    if method == "triofm_f2":       # eq:alphai-f2, i-th diagonal entries (R2)
        return (-(_d(T, U(Q)) + _d(Q, U(T))),
                -(_d(R, U(Q)) + _d(T, U(P.T)) + _d(T, U(P)) + _d(P, U(T))
                  + _d(Q, U(Rp)) + _d(Q, U(R))),
                2.0 * np.diag(T) - (_d(R, U(P.T)) + _d(R, U(P)) + _d(T, U(M))
                                    + _d(P, U(Rp)) + _d(P, U(R)) + _d(Q, U(W))),
                2.0 * np.diag(R) - (_d(R, U(M)) + _d(P, U(W))))
    raise ValueError(method)


@dataclass
class OFMResult:
    X: np.ndarray
    iters: int
    converged: bool
    diverged: bool
    grad_norm0: float
    grad_norm: float
    objective: float
    history: np.ndarray                     # [T, 4] objective, ||G||_F, alpha min, alpha max
    alphas: list = field(default_factory=list)     # per iteration: k-vector
    betas: list = field(default_factory=list)      # per iteration: k-vector (0 at t = 0)
    codes: list = field(default_factory=list)      # per iteration: k branch codes
    state: dict = field(default_factory=dict)      # final AX, M, W (tests)


def run_ofm(op: Operator, method: str, X0, T: int, *, tol=0.0, beta_rule="pr+",
            line_search=True, alpha_fixed=0.0, refresh=1, precision="f64",
            callback=None) -> OFMResult:
    """Algorithm 2 for `T` iterations (T updates of X).

    refresh: 1 = the paper's schedule (A X, X^T X, X^T A X recomputed every
    iteration); R > 1 = recurrence AX += AV diag(alpha) and algebraic
    M, W updates with a recompute every R iterations; 0 = never recompute (R23).
    precision: "f64", or "f32" = fp32 storage of X, AX, G, V, AV with fp64
    Grams / k x k arithmetic.
    callback: optional callable(t) invoked after iteration t (timing only)."""
    if method not in METHODS:
        raise ValueError(method)
    rnd = (lambda a: a) if precision == "f64" else \
        (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    n, k = X0.shape
    fro2 = fro2_A(op)
    X = rnd(np.array(X0, dtype=np.float64))
    AX = apply_A(op, X, precision)
    M = gram(X, X)
    W = gram(X, AX)
    Gp = Vp = gg_prev = None
    hist = np.full((T, 4), np.nan)
    res = OFMResult(X=X, iters=0, converged=False, diverged=False, grad_norm0=np.nan,
                    grad_norm=np.nan, objective=np.nan, history=hist)
    tri = method.startswith("tri")
    for t in range(T):
        if t > 0 and refresh >= 1 and t % refresh == 0:
            AX = apply_A(op, X, precision)
            M = gram(X, X)
            W = gram(X, AX)
        G = rnd(direction(method, X, AX, M, W))            # Alg. 2 l.8
        gg = colsum(G * G)
        gnorm = float(np.sqrt(np.sum(gg)))
        obj = float(objective(method, M, W, fro2))
        hist[t, 0], hist[t, 1] = obj, gnorm
        if t == 0:
            res.grad_norm0 = gnorm
        res.grad_norm, res.objective = gnorm, obj
        if not np.all(np.isfinite(G)):
            res.diverged = True
            break
        if gnorm == 0.0 or (tol > 0.0 and gnorm <= tol * _C_M[method] * np.sqrt(np.trace(M))):
            res.converged = True
            break
        if t == 0 or beta_rule == "zero":                  # Alg. 2 l.4
            beta = np.zeros(k)
            V = -G
        else:                                              # Alg. 2 l.9-10
            beta = beta_pr(G, Gp, gg_prev, beta_rule)
            V = rnd(-G + Vp * beta[None, :])
        res.betas.append(beta.copy())
        AV = apply_A(op, V, precision)
        Q, P, Tm, Rp = grams(V, X, AV)
        if line_search:                                    # Alg. 2 l.11
            c3, c2, c1, c0 = cubic_coefficients(method, Q, P, Tm, Rp, M, W)
            if tri:
                sel = [select_step(float(c3[i]), float(c2[i]), float(c1[i]), float(c0[i]))
                       for i in range(k)]
                alpha = np.array([s[0] for s in sel])
                codes = [s[1] for s in sel]
            else:
                a, code = select_step(float(c3), float(c2), float(c1), float(c0))
                alpha = np.full(k, a)
                codes = [code] * k
        else:
            alpha = np.full(k, float(alpha_fixed))
            codes = [BRANCH["zero"]] * k
        res.alphas.append(alpha.copy())
        res.codes.append(codes)
        hist[t, 2], hist[t, 3] = alpha.min(), alpha.max()
        if BRANCH["diverged"] in codes:
            res.diverged = True
            break
        X = rnd(X + V * alpha[None, :])                    # Alg. 2 l.12
        AX = rnd(AX + AV * alpha[None, :])
        M = M + P.T * alpha[None, :] + alpha[:, None] * P + alpha[:, None] * Q * alpha[None, :]
        W = W + Rp * alpha[None, :] + alpha[:, None] * Rp.T + alpha[:, None] * Tm * alpha[None, :]
        Gp, Vp, gg_prev = G, V, gg
        res.iters = t + 1
        if callback is not None:
            callback(t)
    res.X = X
    res.state = {"AX": AX, "M": M, "W": W}
    return res

"""Oracle: graph -> shifted normalised Laplacian A = L - 2I (TEST INFRASTRUCTURE ONLY).

P:28-31   L = I - D^{-1/2} S D^{-1/2}, S_ij = 1 if i~j else 0, D_ii = sum_j S_ij.
P:48      A = L - 2I, so A = -I - D^{-1/2} S D^{-1/2}:
          A_ii = -1, A_ij = -s_i s_j for j in N(i), s = d^{-1/2}.
Readings (R12, R13): self-loops dropped, multi-edges collapsed
(S is 0/1); an isolated node has s_i = 0, its row of A is -e_i.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class Operator:
    n: int
    row_ptr: np.ndarray      # int64[n+1]
    col: np.ndarray          # int64[nnz], sorted ascending within each row
    deg: np.ndarray          # int64[n]
    s: np.ndarray            # float64[n], d^{-1/2} (0 for isolated)
    n_edges: int             # unique undirected edges kept
    n_self_loops: int
    n_duplicates: int
    S: sp.csr_matrix         # 0/1 pattern (float64)


def build_operator(n, src, dst) -> Operator:
    """Canonical undirected edge set -> CSR pattern of S and s = D^{-1/2}."""
    src = np.asarray(src, dtype=np.int64).ravel()
    dst = np.asarray(dst, dtype=np.int64).ravel()
    if src.shape != dst.shape:
        raise ValueError("src/dst length mismatch")
    if src.size and (src.min() < 0 or dst.min() < 0 or src.max() >= n or dst.max() >= n):
        raise IndexError("edge endpoint outside [0, n)")
    loop = src == dst
    u = np.minimum(src[~loop], dst[~loop])
    v = np.maximum(src[~loop], dst[~loop])
    keys = np.sort(u * np.int64(n) + v)             # S_ij in {0,1}: dedupe
    if keys.size:
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    u, v = keys // n, keys % n
    rows = np.concatenate([u, v])                   # S symmetric (undirected graph)
    cols = np.concatenate([v, u])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    deg = np.bincount(rows, minlength=n).astype(np.int64)   # D_ii = sum_j S_ij
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    s = np.zeros(n, dtype=np.float64)
    nz = deg > 0
    s[nz] = 1.0 / np.sqrt(deg[nz].astype(np.float64))
    S = sp.csr_matrix((np.ones(cols.size), cols, row_ptr), shape=(n, n))
    return Operator(n=n, row_ptr=row_ptr, col=cols, deg=deg, s=s,
                    n_edges=int(keys.size), n_self_loops=int(loop.sum()),
                    n_duplicates=int((~loop).sum() - keys.size), S=S)


def apply_A(op: Operator, Z: np.ndarray, precision: str = "f64") -> np.ndarray:
    """Y = A Z = -Z - s * (S (s * Z)).

    precision="f32": the fp32-storage policy of DESIGN.md (Z is fp32, the row
    sums and the result are fp32 arithmetic with s rounded to fp32); the result
    is returned as float64 holding fp32 values."""
    if precision == "f64":
        Z = np.asarray(Z, dtype=np.float64)
        s = op.s[:, None]
        return -Z - s * (op.S @ (s * Z))
    Z32 = np.asarray(Z, dtype=np.float32)
    s32 = op.s.astype(np.float32)[:, None]
    S32 = op.S.astype(np.float32)
    acc = S32 @ (s32 * Z32)                         # fp32 accumulate
    return ((-Z32) - s32 * acc).astype(np.float32).astype(np.float64)


def dense_A(op: Operator) -> np.ndarray:
    """Dense A for tiny graphs (tests): -I - D^{-1/2} S D^{-1/2}."""
    Sd = op.S.toarray()
    return -np.eye(op.n) - op.s[:, None] * Sd * op.s[None, :]


def fro2_A(op: Operator) -> float:
    """||A||_F^2 = N + sum_i sum_{j in N(i)} (s_i s_j)^2  (diagonal -1 contributes N)."""
    rows = np.repeat(np.arange(op.n), op.deg)
    return float(op.n + np.sum((op.s[rows] * op.s[op.col]) ** 2))

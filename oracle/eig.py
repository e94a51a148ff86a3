"""Oracle: dense cyclic Jacobi eigensolver for tiny symmetric matrices (TEST INFRASTRUCTURE ONLY).

The north star asks the oracle to be checked against "a dense Jacobi
eigendecomposition of L on tiny graphs"; this is the textbook cyclic Jacobi
rotation method (Golub & Van Loan, sec. 8.5), plain loops, fp64.
"""
from __future__ import annotations

import math

import numpy as np


def jacobi_eigh(A, tol=1e-14, max_sweeps=100):
    """Eigenvalues (ascending) and orthonormal eigenvectors (columns) of symmetric A."""
    A = np.array(A, dtype=np.float64)
    n = A.shape[0]
    V = np.eye(n)
    for _ in range(max_sweeps):
        off = math.sqrt(np.sum((A - np.diag(np.diag(A))) ** 2))
        if off <= tol * max(1.0, math.sqrt(np.sum(A * A))):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if apq == 0.0:
                    continue
                tau = (A[q, q] - A[p, p]) / (2.0 * apq)
                t = (1.0 if tau >= 0.0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                # A <- J^T A J with J the (p,q) rotation
                ap = A[:, p].copy()
                aq = A[:, q].copy()
                A[:, p] = c * ap - s * aq
                A[:, q] = s * ap + c * aq
                ap = A[p, :].copy()
                aq = A[q, :].copy()
                A[p, :] = c * ap - s * aq
                A[q, :] = s * ap + c * aq
                vp = V[:, p].copy()
                vq = V[:, q].copy()
                V[:, p] = c * vp - s * vq
                V[:, q] = s * vp + c * vq
    w = np.diag(A).copy()
    order = np.argsort(w, kind="stable")
    return w[order], V[:, order]

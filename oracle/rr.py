"""Oracle: orthogonalisation + Rayleigh-Ritz post-step and the relerr metric
(TEST INFRASTRUCTURE ONLY).

P:596  "After orthogonalizing the results given by OFMs, the Rayleigh-Ritz
        method is applied to the orthogonal vectors to compute the Ritz pairs,
        which serve as the eigenvalues and eigenvectors of the original matrix
        A.  The Rayleigh-Ritz method, including one SpMM, several dot products,
        and an eigendecomposition of a k x k matrix ..."
P:589  relerr = ||B U - U Lambda||_F / ||U Lambda||_F, B "the normalized
        similarity matrix with transition 2 on the diagonal", Lambda, U the
        Ritz pairs.

Readings (R24-R26):
  R24  orthogonalisation = Cholesky-QR of X: M = X^T X = L L^T, Q = X L^{-T}
       (the k x k route that needs no N-length orthogonalisation pass);
  R25  the Rayleigh quotient matrix is formed from the symmetric part of
       W = X^T (A X): H = L^{-1} ((W + W^T)/2) L^{-T};
  R26  B = L + 2I = A + 4I: same eigenvectors as A, Ritz values
       of B are theta + 4, and B U - U (Theta + 4I) = A U - U Theta.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from .eig import jacobi_eigh
from .operator import apply_A


@dataclass
class RRResult:
    theta: np.ndarray     # Ritz values of A, ascending (k)
    U: np.ndarray         # Ritz vectors (n x k), orthonormal columns
    relerr: float         # P:589 with B = A + 4I


def rayleigh_ritz(op, X):
    """Ritz pairs of A on span(X) and relerr, step by step."""
    X = np.asarray(X, dtype=np.float64)
    AX = apply_A(op, X)                           # the one SpMM
    M = X.T @ X                                   # dot products
    W = X.T @ AX
    L = np.linalg.cholesky(M)                     # M = L L^T (raises if X is rank deficient)
    Ws = 0.5 * (W + W.T)
    H = sla.solve_triangular(L, sla.solve_triangular(L, Ws, lower=True).T, lower=True).T
    H = 0.5 * (H + H.T)                           # exact symmetry for the Jacobi sweep
    theta, Z = jacobi_eigh(H)                     # k x k eigendecomposition (ascending)
    T = sla.solve_triangular(L.T, Z, lower=False)  # L^{-T} Z
    U = X @ T                                     # Ritz vectors  Q Z = X L^{-T} Z
    AU = AX @ T                                   # A U (linearity: no second SpMM)
    resid = AU - U * theta[None, :]               # = B U - U (Theta + 4I)
    lam_B = theta + 4.0
    relerr = float(np.linalg.norm(resid) / np.linalg.norm(U * lam_B[None, :]))
    return RRResult(theta=theta, U=U, relerr=relerr)

"""Oracle: row normalisation, Lloyd K-means, ARI, NMI (TEST INFRASTRUCTURE ONLY).

Alg. 1 l.4: "Normalize each row of the feature matrix" (a zero row stays zero).
Alg. 1 l.5 / P:587: Euclidean K-means; ARI (Hubert-Arabie) and NMI.
Readings (R20, R21): Lloyd from GIVEN centroids; squared distance
summed d = 0..dim-1 sequentially in fp64, ties -> lowest centroid index; empty
cluster keeps its centroid; stop when no label changes or after max_iters
assignments; NMI normalised by the arithmetic mean of the entropies.
"""
from __future__ import annotations

import numpy as np


def row_normalize(X):
    X = np.asarray(X, dtype=np.float64)
    nrm = np.sqrt(np.sum(X * X, axis=1))
    out = np.zeros_like(X)
    nz = nrm > 0.0
    out[nz] = X[nz] / nrm[nz, None]
    return out


def _sqdist(Y, C):
    """d2[r, c] = sum_{d=0}^{dim-1} (Y[r,d] - C[c,d])^2, summed in this order."""
    d2 = np.zeros((Y.shape[0], C.shape[0]))
    for d in range(Y.shape[1]):
        diff = Y[:, d, None] - C[None, :, d]
        d2 = d2 + diff * diff
    return d2


def kmeans_lloyd(Y, C0, max_iters=100):
    """Returns (labels int32[n], centroids [K,dim], iterations, inertia)."""
    Y = np.asarray(Y, dtype=np.float64)
    C = np.array(C0, dtype=np.float64)
    K = C.shape[0]
    labels = None
    it = 0
    inertia = np.nan
    for it in range(1, max_iters + 1):
        d2 = _sqdist(Y, C)
        new = np.argmin(d2, axis=1).astype(np.int32)        # first minimum -> lowest index
        inertia = float(np.sum(d2[np.arange(Y.shape[0]), new]))
        if labels is not None and np.array_equal(new, labels):
            break
        labels = new
        cnt = np.bincount(labels, minlength=K)
        for c in range(K):
            if cnt[c] > 0:
                C[c] = Y[labels == c].sum(axis=0) / cnt[c]
    return labels, C, it, inertia


def _comb2(x):
    x = np.asarray(x, dtype=np.float64)
    return x * (x - 1.0) / 2.0


def _contingency(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    if a.size != b.size:
        raise ValueError("length mismatch")
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    C = np.zeros((ai.max() + 1, bi.max() + 1), dtype=np.int64)
    np.add.at(C, (ai, bi), 1)
    return C


def ari(a, b):
    """(sum C(n_ij,2) - E) / (0.5 (sum C(a_i,2) + sum C(b_j,2)) - E),
    E = sum C(a_i,2) sum C(b_j,2) / C(n,2)."""
    C = _contingency(a, b)
    n = C.sum()
    sij = _comb2(C).sum()
    sa = _comb2(C.sum(axis=1)).sum()
    sb = _comb2(C.sum(axis=0)).sum()
    e = sa * sb / _comb2(n) if n > 1 else 0.0
    den = 0.5 * (sa + sb) - e
    if den == 0.0:
        return 1.0
    return float((sij - e) / den)


def nmi(a, b):
    """2 I(U;V) / (H(U) + H(V)), natural log; 1 if both entropies are 0."""
    C = _contingency(a, b).astype(np.float64)
    n = C.sum()
    pa = C.sum(axis=1) / n
    pb = C.sum(axis=0) / n
    ha = -np.sum(pa[pa > 0] * np.log(pa[pa > 0]))
    hb = -np.sum(pb[pb > 0] * np.log(pb[pb > 0]))
    if ha + hb == 0.0:
        return 1.0
    pij = C / n
    nz = pij > 0
    mi = np.sum(pij[nz] * np.log(pij[nz] / (pa[:, None] * pb[None, :])[nz]))
    return float(2.0 * mi / (ha + hb))

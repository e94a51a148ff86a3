"""Seeded degree-corrected SBM graphs, X0 and K-means init rows.

Recipe: SURVEY.md section 8(d).1, restated in DESIGN.md "Input recipe".  The
paper's workloads are the Graph Challenge streaming-SBM graphs,
which are not available here; these synthetic graphs stand in for them with
BASELINE.json's shapes (N, blocks, average degree, within:between ratio,
power-law degree propensities with exponent -2.1 on [10, 100]).

Everything is drawn from numpy's PCG64 with an explicit seed, so both the
oracle and the CUDA path receive bit-identical inputs.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int                  # nodes
    blocks: int             # planted blocks
    edges: int              # unique undirected edges E
    ratio: float            # within:between edge ratio r
    k: int                  # features
    dirichlet: Optional[float]  # None -> equal block sizes, else Dirichlet(alpha)
    seed_graph: int
    seed_x0: int
    seed_km: int
    iters: int              # iteration budget of the config
    kind: str = "dcsbm"     # "dcsbm" or "rmat" (NEXT-3 stress graphs; blocks = K-means clusters)


# BASELINE.json "configs" (c1..c5); seeds from SURVEY 8(d).1.
CONFIGS = {
    "c1": Config("c1", 1_000, 11, 8_000, 3.0, 11, None, 101, 102, 103, 200),
    "c2": Config("c2", 20_000, 32, 160_000, 2.5, 32, 5.0, 201, 202, 203, 500),
    "c3": Config("c3", 200_000, 71, 1_600_000, 5.0, 64, 5.0, 301, 302, 303, 200),
    "c3hi": Config("c3hi", 200_000, 71, 1_600_000, 2.5, 64, 5.0, 311, 302, 303, 200),
    "c4": Config("c4", 5_000_000, 64, 50_000_000, 3.0, 64, 5.0, 401, 402, 403, 50),
    "c5": Config("c5", 1_000_000, 48, 8_000_000, 3.0, 48, 5.0, 501, 502, 503, 500),
    # optional, paper-shaped: the Graph Challenge graphs' nnz(A)/N ~ 48
    # (Table 2) at 1M nodes, equal blocks
    "c6": Config("c6", 1_000_000, 64, 23_700_000, 3.0, 64, None, 601, 602, 603, 50),
    # NEXT-3 stress graph shaped like the paper's Graph500 scaling input (P:510-511,
    # Graph500 R-MAT a,b,c = 0.57, 0.19, 0.19, edge factor 16; k = 8 as in P:642),
    # at scale 22 (4.2M nodes): heavy-tailed degrees, high partition imbalance
    "r22": Config("r22", 1 << 22, 8, 16 << 22, 0.0, 8, None, 701, 702, 703, 50, "rmat"),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _block_sizes(rng, n, blocks, dirichlet):
    if dirichlet is None:
        p = np.full(blocks, 1.0 / blocks)
    else:
        p = rng.dirichlet(np.full(blocks, float(dirichlet)))
    sizes = np.maximum(np.floor(p * n).astype(np.int64), 1)
    sizes[-1] = n - sizes[:-1].sum()
    # keep every block non-empty even if the remainder went negative
    while sizes[-1] < 1:
        j = int(np.argmax(sizes[:-1]))
        sizes[j] -= 1
        sizes[-1] += 1
    return sizes


def _powerlaw(rng, n, gamma=2.1, lo=10.0, hi=100.0):
    """Inverse-CDF draw from pdf ~ x^-gamma on [lo, hi]."""
    a = lo ** (1.0 - gamma)
    b = hi ** (1.0 - gamma)
    u = rng.random(n)
    return (a + u * (b - a)) ** (1.0 / (1.0 - gamma))


def _sorted_unique(k):
    k = np.sort(k)
    if k.size:
        keep = np.empty(k.size, dtype=bool)
        keep[0] = True
        np.not_equal(k[1:], k[:-1], out=keep[1:])
        k = k[keep]
    return k


def _collect_unique(rng, n, target, sampler):
    """Draw candidate pairs until at least `target` unique undirected non-loop
    pairs exist, then keep a uniformly random subset of exactly `target`."""
    keys = np.empty(0, dtype=np.int64)          # sorted, unique
    while keys.size < target:
        need = target - keys.size
        u, v = sampler(int(need * 1.08) + 64)
        ok = u != v
        u, v = u[ok], v[ok]
        k = _sorted_unique(np.minimum(u, v) * np.int64(n) + np.maximum(u, v))
        if keys.size:
            pos = np.searchsorted(keys, k)
            dup = (pos < keys.size) & (keys[np.minimum(pos, keys.size - 1)] == k)
            k = k[~dup]
            keys = np.sort(np.concatenate([keys, k]))
        else:
            keys = k
    if keys.size > target:
        keys = keys[np.sort(rng.permutation(keys.size)[:target])]
    return keys


def dcsbm_graph(n, blocks, edges, ratio, seed, dirichlet=None, gamma=2.1,
                dmin=10.0, dmax=100.0):
    """Return (src int64[E], dst int64[E], labels int32[n]) of a seeded DCSBM.

    Node ids are a random permutation of block order (no hidden locality);
    edge orientation and order are random.  Exactly `edges` unique undirected
    edges, round(E*r/(r+1)) of them within blocks."""
    rng = _rng(seed)
    sizes = _block_sizes(rng, n, blocks, dirichlet)
    block_of_sorted = np.repeat(np.arange(blocks, dtype=np.int32), sizes)
    order = rng.permutation(n).astype(np.int64)       # sorted position -> node id
    labels = np.empty(n, dtype=np.int32)
    labels[order] = block_of_sorted
    theta = _powerlaw(rng, n, gamma, dmin, dmax)      # propensity per sorted position
    cum = np.cumsum(theta)
    total = cum[-1]
    bstart = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    bend = bstart + sizes
    mass_before = np.where(bstart > 0, cum[np.maximum(bstart - 1, 0)], 0.0)
    bmass = cum[bend - 1] - mass_before

    def draw_global(m):
        # sorted uniforms: same distribution, cache-friendly search
        pos = np.searchsorted(cum, np.sort(rng.random(m)) * total, side="right")
        return np.minimum(pos, n - 1)

    def within(m):
        pu = draw_global(m)
        b = block_of_sorted[pu]
        x = mass_before[b] + rng.random(m) * bmass[b]
        pv = np.searchsorted(cum, x, side="right")
        pv = np.clip(pv, bstart[b], bend[b] - 1)
        return order[pu], order[pv]

    def between(m):
        pu = draw_global(m)
        pv = draw_global(m)[rng.permutation(m)]
        ok = block_of_sorted[pu] != block_of_sorted[pv]
        return order[pu[ok]], order[pv[ok]]

    e_w = int(round(edges * ratio / (ratio + 1.0)))
    e_b = edges - e_w
    kw = _collect_unique(rng, n, e_w, within) if e_w > 0 else np.empty(0, np.int64)
    kb = _collect_unique(rng, n, e_b, between) if e_b > 0 else np.empty(0, np.int64)
    keys = np.concatenate([kw, kb])
    keys = keys[rng.permutation(keys.size)]
    u = keys // n
    v = keys % n
    flip = rng.random(keys.size) < 0.5
    src = np.where(flip, v, u).astype(np.int64)
    dst = np.where(flip, u, v).astype(np.int64)
    return src, dst, labels


def rmat_graph(scale, edges, seed, a=0.57, b=0.19, c=0.19):
    """Graph500-style R-MAT edge list (Chakrabarti et al.; Graph500 spec
    parameters): each edge picks one quadrant per level with probabilities
    (a, b, c, 1-a-b-c); node ids are then randomly permuted so the high-degree
    nodes carry no locality.  Self-loops and duplicates are left in (the graph
    build drops / collapses them, R13).  Labels are all zero (no planted blocks)."""
    rng = _rng(seed)
    n = 1 << scale
    u = np.zeros(edges, dtype=np.int64)
    v = np.zeros(edges, dtype=np.int64)
    for lvl in range(scale):
        r = rng.random(edges)
        bit_u = r >= a + b                     # quadrants c, d: lower half for u
        bit_v = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= bit_u.astype(np.int64) << lvl
        v |= bit_v.astype(np.int64) << lvl
    perm = rng.permutation(n).astype(np.int64)
    return perm[u], perm[v], np.zeros(n, dtype=np.int32)


def stream_parts(src, dst, parts, seed):
    """Random permutation of the edges split into `parts` nearly equal parts
    (sizes differ by <= 1), for the edge-sampling streaming protocol."""
    rng = _rng(seed)
    perm = rng.permutation(src.size)
    return [(src[idx], dst[idx]) for idx in np.array_split(perm, parts)]


def snowball_parts(n, src, dst, parts, seed):
    """Snowball-sampling streaming parts ("Streaming Graphs - Snowball
    Sampling"; the paper does not define the procedure, R27 follows
    SPEC S:88): breadth-first search from a seeded random node (restarting from
    the lowest-numbered undiscovered node when a component is exhausted) gives
    every node a discovery rank; an edge is revealed once both endpoints are
    discovered, i.e. edges are ordered by max(rank(u), rank(v)) (ties in the
    input order) and split into `parts` contiguous parts whose sizes differ by
    <= 1.  Input generator only: no method arithmetic."""
    import scipy.sparse as sp
    import scipy.sparse.csgraph as csg
    rng = _rng(seed)
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    A = sp.csr_matrix((np.ones(src.size, dtype=np.int8), (src, dst)), shape=(n, n))
    A = ((A + A.T) > 0).astype(np.int8).tocsr()
    rank = np.full(n, -1, dtype=np.int64)
    nxt = 0
    start = int(rng.integers(n))
    while True:
        order = csg.breadth_first_order(A, start, directed=False, return_predecessors=False)
        order = order[rank[order] < 0]
        rank[order] = np.arange(nxt, nxt + order.size)
        nxt += order.size
        left = np.nonzero(rank < 0)[0]
        if left.size == 0:
            break
        start = int(left[0])
    key = np.maximum(rank[src], rank[dst])
    idx = np.argsort(key, kind="stable")
    return [(src[c], dst[c]) for c in np.array_split(idx, parts)]


def x0_block(n, k, seed, dtype=np.float64):
    """X0 ~ N(0, 1/N) entries: standard normal / sqrt(N)."""
    x = _rng(seed).standard_normal((n, k)) / np.sqrt(n)
    return np.ascontiguousarray(x.astype(dtype))


def kmeans_init_rows(n, n_clusters, seed):
    """K distinct row indices (Forgy init); both sides gather centroids from
    their own features at these rows."""
    return np.sort(_rng(seed).choice(n, size=n_clusters, replace=False)).astype(np.int64)


_CACHE = {}


def config_graph(cfg: Config):
    """Graph of a named config, memoised in-process and (for large configs) in an
    on-disk cache (OFSC_SYNTH_CACHE, default /tmp/ofsc_synth) keyed by all
    generator parameters.  The cache only saves generation time; the arrays are
    a pure function of the config."""
    key = cfg.name
    if key in _CACHE:
        return _CACHE[key]
    path = None
    if cfg.edges >= 1_000_000:
        d = os.environ.get("OFSC_SYNTH_CACHE", "/tmp/ofsc_synth")
        tag = f"{cfg.name}_{cfg.kind}_{cfg.n}_{cfg.blocks}_{cfg.edges}_{cfg.ratio}_{cfg.dirichlet}_{cfg.seed_graph}_v1"
        path = os.path.join(d, tag + ".npz")
        if os.path.exists(path):
            try:
                z = np.load(path)
                _CACHE[key] = (z["src"], z["dst"], z["labels"])
                return _CACHE[key]
            except Exception:
                pass
    if cfg.kind == "rmat":
        out = rmat_graph(int(cfg.n).bit_length() - 1, cfg.edges, cfg.seed_graph)
    else:
        out = dcsbm_graph(cfg.n, cfg.blocks, cfg.edges, cfg.ratio, cfg.seed_graph, cfg.dirichlet)
    if path is not None:
        try:
            os.makedirs(os.path.dirname(path), exist_ok=True)
            tmp = path + f".{os.getpid()}.tmp.npz"
            np.savez(tmp, src=out[0], dst=out[1], labels=out[2])
            os.replace(tmp, path)
        except Exception:
            pass
    _CACHE[key] = out
    return out

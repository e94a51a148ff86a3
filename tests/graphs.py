"""Small named graphs with known spectra (test fixtures; no method arithmetic)."""
import itertools

import numpy as np


def edges(pairs):
    p = np.array(list(pairs), dtype=np.int64).reshape(-1, 2)
    return p[:, 0].copy(), p[:, 1].copy()


def clique(n, off=0):
    return [(off + i, off + j) for i, j in itertools.combinations(range(n), 2)]


def path(n):
    return [(i, i + 1) for i in range(n - 1)]


def cycle(n):
    return [(i, (i + 1) % n) for i in range(n)]


def star(m):
    return [(0, i) for i in range(1, m + 1)]


def complete_bipartite(a, b):
    return [(i, a + j) for i in range(a) for j in range(b)]


def clique_union(sizes):
    out, off = [], 0
    for s in sizes:
        out += clique(s, off)
        off += s
    return out, off


def bridged_cliques(sizes, bridges=1):
    """Cliques chained by `bridges` edges between consecutive cliques."""
    out, off, starts = [], 0, []
    for s in sizes:
        starts.append(off)
        out += clique(s, off)
        off += s
    for a in range(len(sizes) - 1):
        for b in range(bridges):
            out.append((starts[a] + b, starts[a + 1] + b))
    return out, off


def random_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, m), rng.integers(0, n, m)

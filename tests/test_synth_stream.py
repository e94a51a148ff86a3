"""Streaming input generators (harness): edge-sampling and snowball parts."""
import numpy as np

from synth import dcsbm_graph, stream_parts, snowball_parts
from tests import graphs as G


def as_set(parts):
    return sorted(zip(np.concatenate([p[0] for p in parts]).tolist(),
                      np.concatenate([p[1] for p in parts]).tolist()))


def test_parts_are_a_disjoint_union():
    src, dst, _ = dcsbm_graph(2000, 5, 8000, 3.0, 1, 5.0)
    ref = sorted(zip(src.tolist(), dst.tolist()))
    for parts in (stream_parts(src, dst, 10, 2), snowball_parts(2000, src, dst, 10, 3)):
        assert as_set(parts) == ref
        sizes = [p[0].size for p in parts]
        assert max(sizes) - min(sizes) <= 1


def test_snowball_reveals_the_seed_component_first():
    """Two disjoint cliques: every edge of the clique holding the seed comes
    before the first edge of the other clique."""
    pairs, n = G.clique_union([12, 9])
    s, d = G.edges(pairs)
    for seed in range(6):
        parts = snowball_parts(n, s, d, 7, seed)
        seq = np.concatenate([p[0] for p in parts])
        comp = (seq >= 12).astype(int)                 # 0: first clique, 1: second
        first = comp[0]
        switch = np.argmax(comp != first)
        assert np.all(comp[:switch] == first) and np.all(comp[switch:] != first)


def test_snowball_is_bfs_ordered_on_a_path():
    """Path graph: discovery ranks grow along the path from the seed, so the
    revealed edges of every prefix form a connected sub-path containing the seed."""
    n = 50
    s, d = G.edges(G.path(n))
    parts = snowball_parts(n, s, d, 10, 4)
    seen = set()
    for ps, pd in parts:
        seen |= set(ps.tolist()) | set(pd.tolist())
        lo, hi = min(seen), max(seen)
        assert seen == set(range(lo, hi + 1))


def test_rmat_degree_skew_and_shape():
    """R-MAT (NEXT-3 stress input): ids in range, heavy-tailed degrees (max degree
    far above the mean, as in Graph500), deterministic from the seed."""
    from synth import rmat_graph
    s, d, lab = rmat_graph(12, 16 << 12, 3)
    n = 1 << 12
    assert s.min() >= 0 and d.max() < n and lab.shape == (n,)
    deg = np.bincount(np.concatenate([s, d]), minlength=n)
    assert deg.max() > 20 * deg.mean()
    s2, d2, _ = rmat_graph(12, 16 << 12, 3)
    assert np.array_equal(s, s2) and np.array_equal(d, d2)

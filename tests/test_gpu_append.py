"""Incremental CSR merge (ofsc_graph_append; SURVEY 8(f) NEXT-2, P:609 streaming):
after every appended part the graph equals the one built from the cumulative
edge list -- CSR and s bit-exact against the oracle's operator, ||A||_F^2 and
counts equal to a fresh GPU build -- and the iteration on it matches the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator, run_ofm, fro2_A  # noqa: E402
from synth import dcsbm_graph, stream_parts, x0_block  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


def cumulative(parts, i):
    return (np.concatenate([p[0] for p in parts[:i]]), np.concatenate([p[1] for p in parts[:i]]))


def check_equal_to_oracle(g, op, inv=None):
    rp, col, s = g.copy_csr()
    if inv is None:
        assert np.array_equal(rp, op.row_ptr)
        assert np.array_equal(col.astype(np.int64), op.col)
        assert np.array_equal(s, op.s)


@pytest.mark.parametrize("device_edges", [False, True])
def test_append_equals_rebuild(device_edges):
    n = 4000
    src, dst, _ = dcsbm_graph(n, 10, 30000, 3.0, 91, 5.0)
    # duplicates across parts (both orientations) and self-loops in the stream
    src = np.concatenate([src, dst[:500], np.arange(50)])
    dst = np.concatenate([dst, src[:500], np.arange(50)])
    parts = stream_parts(src, dst, 10, 92)
    g = ofsc.Graph(n, *parts[0])
    for i in range(2, 11):
        ps, pd = parts[i - 1]
        if device_edges:
            g.append(torch.from_numpy(ps).cuda(), torch.from_numpy(pd).cuda())
        else:
            g.append(ps, pd)
        cs, cd = cumulative(parts, i)
        op = build_operator(n, cs, cd)
        check_equal_to_oracle(g, op)
        ref = ofsc.Graph(n, cs, cd)
        a, b = g.info, ref.info
        for key in ("n_edges_kept", "nnz_global", "nnz_local", "n_isolated", "max_degree",
                    "n_self_loops_dropped", "n_duplicates_dropped"):
            assert a[key] == b[key], key
        assert a["fro2_A"] == b["fro2_A"]              # same CSR, same kernel: bit-exact
        assert abs(a["fro2_A"] - fro2_A(op)) <= 1e-12 * fro2_A(op)
        ref.close()


def test_append_reordered_graph_keeps_its_order():
    """A reordered graph keeps its community row order; new edges are relabelled
    into it, so the internal CSR is the oracle's operator of the relabelled edges."""
    n = 3000
    src, dst, _ = dcsbm_graph(n, 6, 20000, 3.0, 93, 5.0)
    parts = stream_parts(src, dst, 4, 94)
    g = ofsc.Graph(n, *parts[0], reorder=True)
    perm = g.copy_perm()
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    for i in range(2, 5):
        g.append(*parts[i - 1])
        assert np.array_equal(g.copy_perm(), perm)
        cs, cd = cumulative(parts, i)
        op = build_operator(n, inv[cs], inv[cd])
        check_equal_to_oracle(g, op)


def test_append_edge_cases():
    n = 100
    s0, d0 = np.array([0, 1, 2]), np.array([1, 2, 3])
    g = ofsc.Graph(n, s0, d0)
    info0 = dict(g.info)
    g.append(np.array([], np.int64), np.array([], np.int64))      # empty batch: no-op
    g.append(np.array([1, 5, 5]), np.array([0, 5, 5]))            # duplicate + self-loops only
    assert g.info["n_edges_kept"] == 3 and g.info["nnz_global"] == 6
    assert g.info["n_self_loops_dropped"] == 2 and g.info["n_duplicates_dropped"] == 1
    assert g.info["n_isolated"] == info0["n_isolated"]
    with pytest.raises(ofsc.OfscError) as e:
        g.append(np.array([0, 7]), np.array([n, 8]))              # endpoint out of range
    assert e.value.status == 2
    assert g.info["n_edges_kept"] == 3                            # graph unchanged
    g.append(np.array([98, 97]), np.array([99, 99]))              # isolated nodes join
    op = build_operator(n, np.array([0, 1, 2, 98, 97]), np.array([1, 2, 3, 99, 99]))
    check_equal_to_oracle(g, op)
    assert g.info["n_isolated"] == n - 7


def test_append_out_of_range_on_reordered_graph():
    """A reordered graph relabels the new edges through its permutation; endpoints
    outside [0, n) must be rejected (OFSC_ERR_RANGE) before any lookup, and the
    graph must stay unchanged (no out-of-bounds read of the inverse)."""
    n = 3000
    src, dst, _ = dcsbm_graph(n, 8, 24000, 3.0, 91, 5.0)
    g = ofsc.Graph(n, src[:20000], dst[:20000], reorder=True)
    info0 = dict(g.info)
    rp0, col0, s0 = g.copy_csr()
    for bad_s, bad_d in ((np.array([0, 7]), np.array([n, 8])),
                         (np.array([-1, 7]), np.array([3, 8])),
                         (np.array([5, 2 ** 40]), np.array([6, 9]))):
        with pytest.raises(ofsc.OfscError) as e:
            g.append(bad_s, bad_d)
        assert e.value.status == 2
        assert g.info == info0
        rp, col, s_ = g.copy_csr()
        assert np.array_equal(rp, rp0) and np.array_equal(col, col0) and np.array_equal(s_, s0)
    g.append(src[20000:], dst[20000:])                          # a valid batch still merges
    assert g.info["n_edges_kept"] == 24000


@pytest.mark.parametrize("method", ["ofm_f1", "triofm_f2"])
def test_iteration_on_appended_graph(method):
    """The run workspace is rebuilt after an append: 10 iterations on the
    appended graph match the oracle on the cumulative edges (north-star 1e-10)."""
    n, k = 3000, 8
    src, dst, _ = dcsbm_graph(n, 8, 24000, 3.0, 95, 5.0)
    parts = stream_parts(src, dst, 3, 96)
    g = ofsc.Graph(n, *parts[0])
    X0 = x0_block(n, k, 97)
    X = torch.from_numpy(X0.copy()).cuda()
    ofsc.run(g, method, X, 5)                        # workspace + captured graphs exist
    for i in (2, 3):
        g.append(*parts[i - 1])
    cs, cd = cumulative(parts, 3)
    op = build_operator(n, cs, cd)
    X = torch.from_numpy(X0.copy()).cuda()
    r = ofsc.run(g, method, X, 10)
    o = run_ofm(op, method, X0, 10, refresh=0)
    Xg = X.cpu().numpy()
    assert np.linalg.norm(Xg - o.X) / np.linalg.norm(o.X) <= 1e-10
    assert r.report["iters"] == 10

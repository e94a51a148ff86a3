"""Kernel-level parity (P0): CSR build, SpMM, fused SpMM + Gram, line search.

CUDA path (through the C ABI) vs the oracle on identical seeded inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import (build_operator, apply_A, grams, cubic_coefficients, select_step,  # noqa: E402
                    fro2_A, METHODS, run_ofm)
from synth import CONFIGS, config_graph, dcsbm_graph, x0_block  # noqa: E402
from tests import graphs as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


GRAPHS = {
    "c1": lambda: config_graph(CONFIGS["c1"])[:2] + (CONFIGS["c1"].n,),
    "c2": lambda: config_graph(CONFIGS["c2"])[:2] + (CONFIGS["c2"].n,),
    "messy": lambda: (np.array([0, 1, 1, 2, 3, 3, 5, 9, 9, 7]), np.array([1, 0, 1, 3, 2, 2, 5, 8, 7, 9]), 12),
    "ragged": lambda: dcsbm_graph(1037, 5, 6000, 2.0, 9)[:2] + (1037,),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_csr_bit_exact(name):
    s, d, n = GRAPHS[name]()
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d)
    rp, col, sv = g.copy_csr()
    assert np.array_equal(rp, op.row_ptr)
    assert np.array_equal(col.astype(np.int64), op.col)
    assert np.array_equal(sv, op.s)            # 1/sqrt(d): correctly rounded on both sides
    info = g.info
    assert info["n_edges_kept"] == op.n_edges
    assert info["n_self_loops_dropped"] == op.n_self_loops
    assert info["n_duplicates_dropped"] == op.n_duplicates
    assert info["n_isolated"] == int(np.sum(op.deg == 0))
    assert info["max_degree"] == int(op.deg.max())
    assert abs(info["fro2_A"] - fro2_A(op)) <= 1e-13 * fro2_A(op)


def test_build_from_device_edges_and_errors():
    s, d, n = GRAPHS["c1"]()
    g1 = ofsc.Graph(n, s, d)
    g2 = ofsc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    a, b = g1.copy_csr(), g2.copy_csr()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    with pytest.raises(ofsc.OfscError) as e:
        ofsc.Graph(5, np.array([0, 1]), np.array([1, 5]))
    assert e.value.status == 2
    g0 = ofsc.Graph(4, np.array([], np.int64), np.array([], np.int64))   # no edges: A = -I
    Z = torch.randn(4, 3, dtype=torch.float64, device="cuda")
    assert torch.equal(g0.apply(Z), -Z)


@pytest.mark.parametrize("name", ["c1", "c2", "ragged"])
@pytest.mark.parametrize("k", [1, 11, 32, 48, 64])
def test_spmm_f64(name, k):
    s, d, n = GRAPHS[name]()
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d)
    Z = np.random.default_rng(k).standard_normal((n, k))
    Y = g.apply(torch.from_numpy(Z).cuda()).cpu().numpy()
    Yo = apply_A(op, Z)
    assert np.max(np.abs(Y - Yo)) <= 1e-14 * np.max(np.abs(Yo)) * 4


@pytest.mark.parametrize("variant", ["sval", "sval_pf1", "sval_pf2", "sval_pf3", "packed",
                                     "packed_pf2", "packed_nif8", "packed_nif4", "plain_pf2",
                                     "plain_pf3", "heavy", "reorder", "k80", "f32_sval",
                                     "f32_packed"])
def test_spmm_production_variants(variant, monkeypatch):
    """ofsc_graph_apply runs the iteration's SpMM kernel (k_spmm) on KP-padded copies:
    P0 parity of the variants the iteration uses -- the per-nonzero s_j stream (on by
    default above 2e7 nonzeros, forced here), its L2-prefetch forms (OFSC_SPMM_PF),
    degree binning of heavy rows (threshold forced low), the LPA-reordered operator,
    fp32 -- and the plain kernel for k > 64."""
    s, d, n = GRAPHS["c2"]()
    op = build_operator(n, s, d)
    k = 80 if variant == "k80" else 64
    if variant.startswith("sval") or variant == "f32_sval":
        monkeypatch.setenv("OFSC_SPMM_SVAL", "1")
    if variant.startswith("packed") or variant == "f32_packed":
        monkeypatch.setenv("OFSC_SPMM_SVAL", "2")
    if variant == "packed_pf2":
        monkeypatch.setenv("OFSC_SPMM_PF", "2")
    if variant.startswith("packed_nif"):
        monkeypatch.setenv("OFSC_SPMM_PF", "2")
        monkeypatch.setenv("OFSC_SPMM_NIF", variant[-1])
    for pf in ("1", "2", "3"):
        if variant == "sval_pf" + pf:
            monkeypatch.setenv("OFSC_SPMM_PF", pf)
        if variant == "plain_pf" + pf:
            monkeypatch.setenv("OFSC_SPMM_PF_SMALL", pf)
    if variant == "heavy":
        monkeypatch.setenv("OFSC_HEAVY_THRESH", "24")
    g = ofsc.Graph(n, s, d, reorder=(variant == "reorder"))
    Z = np.random.default_rng(5).standard_normal((n, k))
    if variant in ("f32_sval", "f32_packed"):
        Z32 = Z.astype(np.float32)
        Y = g.apply(torch.from_numpy(Z32).cuda()).double().cpu().numpy()
        Yo = oracle_apply_f32(op, Z32)
        assert np.max(np.abs(Y - Yo)) <= 1e-6 * np.max(np.abs(Yo))
        return
    Y = g.apply(torch.from_numpy(Z).cuda()).cpu().numpy()
    Yo = apply_A(op, Z)
    assert np.max(np.abs(Y - Yo)) <= 4e-14 * np.max(np.abs(Yo))


def oracle_apply_f32(op, Z32):
    return apply_A(op, Z32.astype(np.float64), "f32")


@pytest.mark.parametrize("name", ["c1", "c2", "ragged"])
@pytest.mark.parametrize("k", [3, 11, 16, 32, 48, 64])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fused_spmm_gram(name, k, dtype):
    s, d, n = GRAPHS[name]()
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d)
    rng = np.random.default_rng(100 + k)
    Z = rng.standard_normal((n, k)) / np.sqrt(n)
    X = rng.standard_normal((n, k)) / np.sqrt(n)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    if dtype == "f32":
        Z = Z.astype(np.float32).astype(np.float64)
        X = X.astype(np.float32).astype(np.float64)
    Y, Gm = g.apply_gram(torch.from_numpy(Z).to(tdt).cuda(), torch.from_numpy(X).to(tdt).cuda())
    Y = Y.double().cpu().numpy()
    Gm = Gm.cpu().numpy()
    prec = "f64" if dtype == "f64" else "f32"
    Yo = apply_A(op, Z, prec)
    Q, P, T, Rp = grams(Z, X, Yo)
    if dtype == "f64":
        assert np.max(np.abs(Y - Yo)) <= 4e-14 * np.max(np.abs(Yo))
        tol = 1e-13
    else:
        assert np.max(np.abs(Y - Yo)) <= 1e-6 * np.max(np.abs(Yo))
        tol = 1e-6
    for got, want in zip(Gm, (Q, P, T, Rp)):
        assert rel(got, want) <= tol


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("seed", range(6))
def test_line_search_kernel_matches_oracle(method, seed):
    """The k x k kernel on oracle Grams: same alpha (to rounding) and same branch codes."""
    s, d, n = GRAPHS["c1"]()
    op = build_operator(n, s, d)
    rng = np.random.default_rng(seed)
    k = 11
    X = rng.standard_normal((n, k)) / np.sqrt(n) * (1 + seed)
    V = rng.standard_normal((n, k)) / np.sqrt(n) * 10.0 ** (-seed)
    AX, AV = apply_A(op, X), apply_A(op, V)
    Q, P, T, Rp = grams(V, X, AV)
    M, W = X.T @ X, X.T @ AX
    alpha, codes, Mo, Wo = ofsc.line_search(method, Q, P, T, Rp, M, W)
    c3, c2, c1, c0 = cubic_coefficients(method, Q, P, T, Rp, M, W)
    if method.startswith("tri"):
        want = [select_step(c3[i], c2[i], c1[i], c0[i]) for i in range(k)]
    else:
        want = [select_step(c3, c2, c1, c0)] * k
    wa = np.array([w[0] for w in want])
    assert list(codes) == [w[1] for w in want]
    assert np.max(np.abs(alpha - wa)) <= 1e-11 * max(1.0, np.max(np.abs(wa)))
    D = np.diag(alpha)
    assert rel(Mo, M + P.T @ D + D @ P + D @ Q @ D) <= 1e-13
    assert rel(Wo, W + Rp @ D + D @ Rp.T + D @ T @ D) <= 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_line_search_negative_leading_coefficient(seed):
    """TriOFM-f2 columns whose cubic has c3 < 0: the device takes the
    same root as the oracle (one real root: that root; three: the middle one, the
    only local minimum of psi).  Grams are drawn directly (kernel-level hook) with
    an indefinite T so that some c3_i < 0, including a k = 1 textbook case
    (Q = 1, T = 1, P = M = W = 0, R' = r: c3 = -2, c2 = -3r, c1 = 2, c0 = 2r)."""
    rng = np.random.default_rng(900 + seed)
    if seed == 0:
        k = 1
        Q, T = np.ones((1, 1)), np.ones((1, 1))
        P, M, W = np.zeros((1, 1)), np.zeros((1, 1)), np.zeros((1, 1))
        Rp = np.full((1, 1), 0.1)
    else:
        k = 9
        B = rng.standard_normal((40, k))
        Q = B.T @ B / 40
        S = rng.standard_normal((k, k))
        T = (S + S.T) / 2
        P, Rp = rng.standard_normal((k, k)) * 0.3, rng.standard_normal((k, k)) * 0.3
        C = rng.standard_normal((30, k))
        M = C.T @ C / 30
        W = -(M + 0.1 * np.eye(k))
    c3, c2, c1, c0 = cubic_coefficients("triofm_f2", Q, P, T, Rp, M, W)
    assert np.any(np.asarray(c3) < 0)
    alpha, codes, _, _ = ofsc.line_search("triofm_f2", Q, P, T, Rp, M, W)
    want = [select_step(c3[i], c2[i], c1[i], c0[i]) for i in range(k)]
    assert list(codes) == [w[1] for w in want]
    wa = np.array([w[0] for w in want])
    assert np.max(np.abs(alpha - wa)) <= 1e-11 * max(1.0, np.max(np.abs(wa)))


def test_line_search_textbook_cubics_on_device():
    """Grams built so the OFM-f1 cubic is a^3 - a: k = 1, Q = 1, P = 0, T = -1, R' = 0, M = 0."""
    one = np.ones((1, 1))
    zero = np.zeros((1, 1))
    alpha, codes, _, _ = ofsc.line_search("ofm_f1", one, zero, -one, zero, zero, zero)
    assert alpha[0] == -1.0 and codes[0] in (8, 9, 10)
    alpha, codes, _, _ = ofsc.line_search("ofm_f1", zero, zero, zero, zero, zero, zero)
    assert alpha[0] == 0.0 and codes[0] == 0


@pytest.mark.parametrize("name", ["c2", "ragged"])
def test_reordered_graph_is_a_permutation_of_the_operator(name):
    """LPA locality reordering: internal CSR = P S P^T, perm is a permutation,
    communities capture most edges, and the hooks take/return original order."""
    s, d, n = GRAPHS[name]()
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d, reorder=True)
    info = g.info
    perm = g.copy_perm()
    assert info["reordered"] == 1 and np.array_equal(np.sort(perm), np.arange(n))
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rp, col, sv = g.copy_csr()
    assert np.array_equal(sv, op.s[perm])
    for i in np.random.default_rng(0).choice(n, 50, replace=False):
        got = np.sort(perm[col[rp[i]:rp[i + 1]]])
        want = op.col[op.row_ptr[perm[i]]:op.row_ptr[perm[i] + 1]]
        assert np.array_equal(got, want)
    if name == "c2":
        assert info["intra_edge_fraction"] > 0.5 and info["n_communities"] < n // 10
    k = 32
    Z = np.random.default_rng(5).standard_normal((n, k)) / np.sqrt(n)
    X = np.random.default_rng(6).standard_normal((n, k)) / np.sqrt(n)
    Y = g.apply(torch.from_numpy(Z).cuda()).cpu().numpy()
    Yo = apply_A(op, Z)
    assert np.max(np.abs(Y - Yo)) <= 4e-14 * np.max(np.abs(Yo))
    Y2, Gm = g.apply_gram(torch.from_numpy(Z).cuda(), torch.from_numpy(X).cuda())
    Q, P, T, Rp = grams(Z, X, Yo)
    assert np.max(np.abs(Y2.cpu().numpy() - Yo)) <= 4e-14 * np.max(np.abs(Yo))
    for got, want in zip(Gm.cpu().numpy(), (Q, P, T, Rp)):
        assert rel(got, want) <= 1e-13


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("reorder", [False, True])
def test_multirank_layout_with_local_comms(p, reorder):
    """p ranks emulated in one process (local test communicators, no NCCL): each
    rank's graph holds the nnz-balanced row block with slot-remapped columns;
    per-rank SpMM rows and rank-partial Grams reassemble the global results."""
    s, d, n = GRAPHS["c2"]()
    op = build_operator(n, s, d)
    k = 32
    rng = np.random.default_rng(11)
    Z = rng.standard_normal((n, k)) / np.sqrt(n)
    X = rng.standard_normal((n, k)) / np.sqrt(n)
    Yo = apply_A(op, Z)
    want = grams(Z, X, Yo)
    Gsum = np.zeros((4, k, k))
    covered = np.zeros(n, np.int64)
    for r in range(p):
        comm = ofsc.LocalComm(p, r)
        g = ofsc.Graph(n, s, d, comm=comm, reorder=reorder)
        info = g.info
        rb, re_ = info["row_begin"], info["row_end"]
        perm = g.copy_perm()
        if not reorder:
            assert np.array_equal(ofsc.partition_rows(op.row_ptr, p)[[r, r + 1]], [rb, re_])
        nodes = perm[rb:re_]                       # original ids of this rank's rows
        covered[nodes] += 1
        rp, col, _ = g.copy_csr()
        for i in np.random.default_rng(r).choice(re_ - rb, 20, replace=False):
            got = np.sort(perm[col[rp[i]:rp[i + 1]]])
            u = nodes[i]
            assert np.array_equal(got, op.col[op.row_ptr[u]:op.row_ptr[u + 1]])
        Y = g.apply(torch.from_numpy(Z).cuda()).cpu().numpy()      # local rows, internal order
        assert np.max(np.abs(Y - Yo[nodes])) <= 4e-14 * np.max(np.abs(Yo))
        Xl = torch.from_numpy(np.ascontiguousarray(X[nodes])).cuda()
        Y2, Gm = g.apply_gram(torch.from_numpy(Z).cuda(), Xl)
        assert np.max(np.abs(Y2.cpu().numpy() - Yo[nodes])) <= 4e-14 * np.max(np.abs(Yo))
        Gsum += Gm.cpu().numpy()
        with pytest.raises(ofsc.OfscError):
            ofsc.run(g, "ofm_f2", Xl.clone(), 2)       # iterations need real collectives
        g.close()
        comm.close()
    assert np.all(covered == 1)
    for got, w in zip(Gsum, want):
        assert rel(got, w) <= 1e-13


@pytest.mark.parametrize("p", [2, 3, 8])
@pytest.mark.parametrize("reorder", [False, True])
def test_halo_exchange_plan_is_consistent(p, reorder):
    """Halo layout (p > 1): every rank's receive list from q is exactly q's send
    list to it (same rows, same order), the halo is the set of remote columns
    of the rank's rows, and with reordering the halo shrinks (communities stay
    on one rank).  The grouped ncclSend/ncclRecv of the iteration moves exactly
    these rows, so this is the exchange's correctness condition."""
    s, d, n = GRAPHS["c2"]()
    plans, halos = {}, {}
    for r in range(p):
        comm = ofsc.LocalComm(p, r)
        g = ofsc.Graph(n, s, d, comm=comm, reorder=reorder)
        info = g.info
        rb, re_ = info["row_begin"], info["row_end"]
        sc, sg, rc, rg = g.exchange_plan()
        assert sc[r] == 0 and rc[r] == 0 and sc.sum() == info["send_rows"] and rc.sum() == info["halo_rows"]
        rp, col, _ = g.copy_csr()                  # global (internal-order) column ids
        remote = np.unique(col[(col < rb) | (col >= re_)])
        assert np.array_equal(rg, remote)
        plans[r] = (np.concatenate([[0], np.cumsum(sc)]), sg, np.concatenate([[0], np.cumsum(rc)]), rg)
        halos[r] = remote.size
        g.close()
        comm.close()
    for q in range(p):
        for r in range(p):
            if q == r:
                continue
            so, sg = plans[q][0], plans[q][1]
            ro, rg = plans[r][2], plans[r][3]
            assert np.array_equal(sg[so[r]:so[r + 1]], rg[ro[q]:ro[q + 1]]), (q, r)
    if reorder:
        assert sum(halos.values()) < 0.9 * (p - 1) * n     # far below an all-gather


def _heavy_graph():
    """A power-law stress graph: a hub of degree 9,000 (> kHeavyThresh = 256,
    so it is split into 512-neighbour chunks), two hubs of ~5,000 and an R-MAT
    background."""
    from synth import rmat_graph
    rs, rd, _ = rmat_graph(13, 6 << 13, 5)
    n = 1 << 13
    hub = [np.zeros(9000, np.int64), np.arange(1, 9001) % n]
    hub2 = [np.full(5000, 17, np.int64), (np.arange(5000) * 7 + 3) % n]
    hub3 = [np.full(5000, 4242, np.int64), (np.arange(5000) * 11 + 5) % n]
    s = np.concatenate([rs, hub[0], hub2[0], hub3[0]])
    d = np.concatenate([rd, hub[1], hub2[1], hub3[1]])
    return s, d, n


@pytest.mark.parametrize("thresh", [None, 8])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_heavy_rows_split_spmm(thresh, dtype, monkeypatch):
    """Degree-aware row binning: rows above the threshold are summed in chunks
    (fixed chunk order) -- SpMM + Grams match the oracle; thresh = 8 forces most
    rows of the graph through the chunked path."""
    if thresh is not None:
        monkeypatch.setenv("OFSC_HEAVY_THRESH", str(thresh))
    s, d, n = _heavy_graph()
    op = build_operator(n, s, d)
    assert op.deg.max() > 4096
    g = ofsc.Graph(n, s, d)
    k = 32
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((n, k)) / np.sqrt(n)
    X = rng.standard_normal((n, k)) / np.sqrt(n)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    Y, Gm = g.apply_gram(torch.from_numpy(Z).to(tdt).cuda(), torch.from_numpy(X).to(tdt).cuda())
    if dtype == "f64":
        Yo = apply_A(op, Z)
        assert np.max(np.abs(Y.cpu().numpy() - Yo)) <= 4e-14 * np.max(np.abs(Yo))
        assert rel(Gm.cpu().numpy()[2], (Z.T @ Yo)) <= 1e-13
    else:
        Z32 = Z.astype(np.float32).astype(np.float64)
        Yo = apply_A(op, Z32, "f32")
        assert np.max(np.abs(Y.cpu().double().numpy() - Yo)) <= 1e-5 * np.max(np.abs(Yo))
    g.close()


@pytest.mark.parametrize("method", METHODS)
def test_heavy_rows_iteration(method):
    """P2 on the power-law stress graph (hub rows split): 10 iterations vs the oracle."""
    s, d, n = _heavy_graph()
    op = build_operator(n, s, d)
    g = ofsc.Graph(n, s, d, reorder=True)
    X0 = x0_block(n, 8, 31)
    o = run_ofm(op, method, X0, 10, refresh=0)
    X = torch.from_numpy(X0.copy()).cuda()
    r = ofsc.run(g, method, X, 10)
    assert r.report["iters"] == o.iters
    assert rel(X.cpu().numpy(), o.X) <= 1e-10
    g.close()

"""Rayleigh-Ritz post-step parity:
ofsc_rayleigh_ritz (C ABI) against oracle.rr.rayleigh_ritz on identical inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator, run_ofm  # noqa: E402
from oracle.rr import rayleigh_ritz  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402
from tests import graphs as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


def compare(theta, U, rel, o, gap_tol=1e-6):
    scale = np.max(np.abs(o.theta))
    assert np.max(np.abs(theta - o.theta)) <= 1e-12 * scale
    assert abs(rel - o.relerr) <= 1e-12 + 1e-8 * o.relerr
    # Ritz vectors: unique up to sign where the Ritz value is isolated
    k = len(theta)
    for j in range(k):
        gap = min([abs(o.theta[j] - o.theta[i]) for i in range(k) if i != j] or [np.inf])
        if gap <= gap_tol * max(scale, 1.0):
            continue
        sg = np.sign(U[:, j] @ o.U[:, j])
        assert np.max(np.abs(U[:, j] * sg - o.U[:, j])) <= 1e-9 / min(gap, 1.0) * max(scale, 1.0)
    assert np.allclose(U.T @ U, np.eye(k), atol=1e-12)


@pytest.mark.parametrize("name,iters", [("c1", 0), ("c1", 60), ("c2", 30)])
@pytest.mark.parametrize("reorder", [False, True])
def test_rr_matches_oracle(name, iters, reorder):
    cfg = CONFIGS[name]
    s, d, _ = config_graph(cfg)
    op = build_operator(cfg.n, s, d)
    X = x0_block(cfg.n, cfg.k, cfg.seed_x0)
    if iters:
        X = run_ofm(op, "ofm_f2", X, iters, refresh=0).X
    o = rayleigh_ritz(op, X)
    g = ofsc.Graph(cfg.n, s, d, reorder=reorder)
    theta, U, rel = ofsc.rayleigh_ritz(g, torch.from_numpy(X.copy()).cuda())
    compare(theta, U.cpu().numpy(), rel, o)


@pytest.mark.parametrize("k", [1, 5, 17, 33, 64])
def test_rr_widths_ragged(k):
    """Every padded width (16/32/48/64) and k = 1 on a ragged row count."""
    n = 1037
    s, d = G.random_graph(n, 6 * n, 7)
    op = build_operator(n, s, d)
    X = np.random.default_rng(k).standard_normal((n, k))
    o = rayleigh_ritz(op, X)
    g = ofsc.Graph(n, s, d)
    theta, U, rel = ofsc.rayleigh_ritz(g, torch.from_numpy(X.copy()).cuda())
    compare(theta, U.cpu().numpy(), rel, o)


def test_rr_clique_union_and_rank_deficient():
    pairs, n = G.clique_union([5, 7, 4])
    s, d = G.edges(pairs)
    g = ofsc.Graph(n, s, d)
    X = np.zeros((n, 3))
    X[:5, 0], X[5:12, 1], X[12:, 2] = 1, 1, 1
    theta, U, rel = ofsc.rayleigh_ritz(g, torch.from_numpy(X).cuda())
    assert np.allclose(theta, -2.0, atol=1e-13) and rel <= 1e-13
    with pytest.raises(ofsc.OfscError) as e:
        ofsc.rayleigh_ritz(g, torch.ones((n, 2), dtype=torch.float64).cuda())
    assert e.value.status == 2                   # OFSC_ERR_RANGE


def test_rr_f32_storage():
    """fp32 features: X rounded to fp32 on both sides, fp64 arithmetic (tolerance 1e-5)."""
    cfg = CONFIGS["c1"]
    s, d, _ = config_graph(cfg)
    op = build_operator(cfg.n, s, d)
    X = x0_block(cfg.n, cfg.k, cfg.seed_x0).astype(np.float32)
    o = rayleigh_ritz(op, X.astype(np.float64))
    g = ofsc.Graph(cfg.n, s, d)
    theta, U, rel = ofsc.rayleigh_ritz(g, torch.from_numpy(X.copy()).cuda())
    assert U.dtype == torch.float32
    assert np.max(np.abs(theta - o.theta)) <= 1e-5
    assert abs(rel - o.relerr) <= 1e-5 * o.relerr

"""Library memory management (not a paper step): buffers of destroyed graphs are
reused by the next graph of the same shape, and ofsc_trim_memory hands them back
(the device's free memory grows again) without breaking later calls."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from synth import CONFIGS, config_graph, x0_block  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


def _run_once(cfg, s, d, X0):
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    X = torch.from_numpy(X0).cuda()
    r = ofsc.run(g, "ofm_f2", X, 5)
    g.close()
    return X.cpu().numpy(), r.history


def test_reuse_and_trim_are_transparent():
    cfg = CONFIGS["c3"]
    s, d, _ = config_graph(cfg)
    X0 = x0_block(cfg.n, cfg.k, cfg.seed_x0)
    Xa, ha = _run_once(cfg, s, d, X0)
    free0 = torch.cuda.mem_get_info()[0]
    Xb, hb = _run_once(cfg, s, d, X0)          # same shapes: cached blocks reused
    assert np.array_equal(Xa, Xb) and np.array_equal(ha, hb)
    ofsc.trim_memory()
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 > free0                        # the workspace and CSR went back
    Xc, hc = _run_once(cfg, s, d, X0)          # fresh allocations after the trim
    assert np.array_equal(Xa, Xc) and np.array_equal(ha, hc)

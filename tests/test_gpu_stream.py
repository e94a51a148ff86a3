"""Streaming protocol (config c5 shape at small N): snapshots of
cumulative edge parts, each run warm-started from the previous features and
stopped at the gradient tolerance (R14).  GPU vs oracle from the same warm start."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2305_10356_b200 as ofsc  # noqa: E402
from oracle import build_operator, run_ofm  # noqa: E402
from synth import dcsbm_graph, stream_parts, x0_block  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ofsc.lib()


@pytest.mark.parametrize("method", ["ofm_f1", "ofm_f2"])
def test_warm_started_snapshots_match_oracle(method):
    n, k = 3000, 8
    s, d, lab = dcsbm_graph(n, 8, 24000, 3.0, 77, 5.0)
    parts = stream_parts(s, d, 5, 78)
    X = x0_block(n, k, 79)
    iters = []
    for i in range(1, 6):
        ss = np.concatenate([p[0] for p in parts[:i]])
        dd = np.concatenate([p[1] for p in parts[:i]])
        op = build_operator(n, ss, dd)
        g = ofsc.Graph(n, ss, dd, reorder=True)
        Xg = torch.from_numpy(X.copy()).cuda()
        r = ofsc.run(g, method, Xg, 3000, tol=1e-4, check_every=1)
        o = run_ofm(op, method, X, 3000, tol=1e-4, refresh=0)
        assert r.report["converged"] == 1 and o.converged
        # 100+ step trajectories agree only to rounding amplification (R22): the
        # step at which the tolerance is met may move a little, and at a 1e-4
        # gradient tolerance the clustered trailing directions are not yet fixed;
        # the objective agrees
        assert abs(r.report["iters"] - o.iters) <= max(3, 0.2 * o.iters)
        Xn = Xg.cpu().numpy()
        assert abs(r.report["objective"] - o.objective) <= 1e-6 * abs(o.objective)
        iters.append(r.report["iters"])
        X = Xn                                        # warm start for the next snapshot
    # warm starts converge faster than the cold first snapshot
    assert min(iters[2:]) < iters[0]

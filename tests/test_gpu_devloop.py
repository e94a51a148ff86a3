"""Device-side iteration loop (CUDA graph WHILE node, OFSC_DEVLOOP=1): same
iterates, stop step and history as the host-driven loop, in a subprocess so the
environment switch is read fresh."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r'''
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2305_10356_b200 as ofsc
from synth import CONFIGS, config_graph, x0_block
cfg = CONFIGS["c1"]
s, d, _ = config_graph(cfg)
g = ofsc.Graph(cfg.n, s, d)
out = {}
for tol in (1e-6, 0.0):
    X = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    r = ofsc.run(g, "ofm_f1", X, 300, tol=tol, check_every=1, timing_skip=5)
    out[str(tol)] = {"X": X.cpu().numpy().tolist(), "iters": r.report["iters"],
                     "conv": r.report["converged"], "hist": np.nan_to_num(r.history).tolist()}
print(json.dumps(out))
''' % ROOT


def _run(devloop):
    env = dict(os.environ)
    env.pop("OFSC_DEVLOOP", None)
    if devloop:
        env["OFSC_DEVLOOP"] = "1"
    p = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_device_loop_matches_host_loop():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b = _run(False), _run(True)
    for tol in a:
        assert a[tol]["iters"] == b[tol]["iters"] and a[tol]["conv"] == b[tol]["conv"]
        assert a[tol]["X"] == b[tol]["X"]                 # bitwise: same kernels, same order
        assert a[tol]["hist"] == b[tol]["hist"]
    assert a["1e-06"]["conv"] == 1 and a["1e-06"]["iters"] < 300

timeout 900 python -m pytest tests/test_gpu_iterate.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "p1 or p2 or refresh or p5" > gpurun_out/exp15_tests.log 2>&1; tail -2 gpurun_out/exp15_tests.log
python - > gpurun_out/exp15_refresh.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, '.')
import torch, paper_2305_10356_b200 as ofsc
from synth import CONFIGS, config_graph, x0_block
for name in ("c4", "c5"):
    cfg = CONFIGS[name]; s, d, _ = config_graph(cfg)
    g = ofsc.Graph(cfg.n, s, d, reorder=True)
    X0 = torch.from_numpy(x0_block(cfg.n, cfg.k, cfg.seed_x0)).cuda()
    for rep in range(3):
        X = X0.clone(); r = ofsc.run(g, "ofm_f2", X, 12, timing_skip=2, refresh=1)
        X2 = X0.clone(); r2 = ofsc.run(g, "ofm_f2", X2, 12, timing_skip=2, refresh=1, profile=True)
        km = r2.report["kernel_ms"]
        print(json.dumps({"config": name, "ms_per_iter_refresh1": r.report["timed_ms"] / 10, "kernel_ms": [round(v / 10, 3) for v in km], "checksum": float(X.double().sum())}), flush=True)
    g.close()
PY

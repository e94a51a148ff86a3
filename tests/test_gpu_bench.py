"""bench.py's JSON line keeps the driver's contract (keys, types, consistency), run on
a small config on the GPU: the default arm and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_bench(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run_bench("--config", "c2", "--steps", "5", "--warmup", "3", "--passes", "2",
                  "--no-methods", "--no-random-ids", "--e2e-steps", "1")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["unit"] == "it/s" and d["higher_is_better"] is True
    assert abs(d["value"] - 1e3 / d["ms_per_step"]) <= 5e-3 * d["value"]   # rounding of ms_per_step
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] < 1.5 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    kr = d["kernel_rooflines"]
    for name in ("spmm", "update_direction", "direction_gram", "gram_stream"):
        assert 0 < kr[name]["hbm_frac"] < 1.5 and 0 <= kr[name]["fp64_tensor_frac"] < 1.5
        assert kr[name]["binding"] in ("hbm", "fp64_tensor")
    assert d["clustering"]["seeds"] == 10 and -1 <= d["clustering"]["ari_mean"] <= 1


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "c2", "--steps", "3", "--warmup", "1")
    assert d["impl"] == "reference" and d["unit"] == "it/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]

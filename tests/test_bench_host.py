"""Host-side arithmetic of bench.py's roofline objects (no GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_kernel_rooflines_counts():
    n, k, es = 100000, 8, 8
    algo = bench.algorithmic_bytes(n, 5000, n, k, es)
    kern = {name: {"ms_total": 1.0, "launches": 1}
            for name in ("spmm", "update_direction", "direction_gram", "gram_stream")}
    kr = bench.kernel_rooflines(kern, algo, n, k, "ofm_f2", 1000.0)
    B = n * k * es
    # 1 ms per launch: GB/s = bytes / 1e6
    assert abs(kr["update_direction"]["hbm_gbs"] - 8 * B / 1e6) < 0.051
    assert abs(kr["direction_gram"]["hbm_gbs"] - 4 * B / 1e6) < 0.051
    # OFM-f2 C3: two full products; Grams: one symmetric (upper incl. diagonal) + one full
    assert kr["update_direction"]["algorithmic_flops"] == 2 * (2 * n * k * k)
    assert kr["direction_gram"]["algorithmic_flops"] == n * k * (k + 1) + 2 * n * k * k
    tri = bench.kernel_rooflines(kern, algo, n, k, "triofm_f1", 1000.0)
    assert tri["update_direction"]["algorithmic_flops"] == n * k * (k + 1)
    # the f1 methods' C2b forms only diag T, diag R' (no tensor products): HBM-bound 3B
    assert tri["gram_stream"]["algorithmic_flops"] == 0 and tri["gram_stream"]["binding"] == "hbm"
    assert abs(tri["gram_stream"]["hbm_gbs"] - 3 * B / 1e6) < 0.051
    assert kr["gram_stream"]["algorithmic_flops"] == n * k * (k + 1) + 2 * n * k * k
    assert kr["spmm"]["binding"] == "hbm" and kr["spmm"]["fp64_tensor_frac"] == 0.0
    assert kr["fp64_tensor_peak_tflops"] > 30
    # at a power-capped SM clock the DMMA pipe peaks proportionally lower
    kc = bench.kernel_rooflines(kern, algo, n, k, "ofm_f2", 1000.0, 1965.0 / 2)
    assert abs(kc["fp64_tensor_peak_at_sm_clock_tflops"] - kc["fp64_tensor_peak_tflops"] / 2) < 0.01
    assert abs(kc["gram_stream"]["fp64_tensor_frac_at_clock"]
               - 2 * kc["gram_stream"]["fp64_tensor_frac"]) < 1e-3

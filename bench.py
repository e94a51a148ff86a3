#!/usr/bin/env python
"""Benchmark: OF-method iterations/s and HBM GB/s on B200 (BASELINE.json metric).

A "step" is one iteration of Algorithm 2 on the whole graph: the
fused chain C3 (update + direction) -> beta -> C4 (direction + Q, P Grams) ->
[all-gather V] -> C2 (SpMM + T, R' Grams) -> Gram reduce -> [all-reduce] ->
exact line search.  Workload: BASELINE config c4 (DCSBM N = 5M, 50M edges,
k = 64, fp64), rows partitioned over N GPUs (strong scaling on the same graph).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value`  = K / (max over ranks of the CUDA-event time of the K iterations).
`e2e`    = the same metric through ofsc_spectral_cluster (C ABI, Algorithm 1
           end to end) from pinned HOST buffers: edge upload + graph build +
           T_e2e iterations + row normalise + K-means + feature/label download.
`roofline` = the dominant kernel's algorithmic bytes per launch / its average
           CUDA-event duration (profiled pass on the same stream), vs the
           measured HBM copy peak (MEASURED_PEAKS.json).
`cpu_baseline` = the oracle (numpy/scipy, as it stands) on the host cores.
The reference arm (--impl reference) times the oracle the same way.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, config_graph, x0_block, kmeans_init_rows  # noqa: E402

METRIC = "OF-method iterations/sec and HBM GB/s (fraction of peak) at 1/2/4/8 B200"
PHASES = ("update_direction", "beta", "direction_gram", "spmm", "gram_reduce",
          "line_search", "refresh", "comm", "gram_stream", "unused")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--method", default="ofm_f2")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--refresh", type=int, default=0)
    ap.add_argument("--reorder", type=int, default=1, help="1: LPA locality reordering of the rows")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-methods", action="store_true")
    ap.add_argument("--passes", type=int, default=5, help="timed passes of K steps (median, min)")
    ap.add_argument("--no-random-ids", action="store_true")
    ap.add_argument("--no-ari", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check: each rank prints its rank / world size and exits")
    return ap.parse_args()


def launch_ranks(args):
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one process per
    GPU, torch.distributed.run on 127.0.0.1).  Inside torchrun WORLD_SIZE must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus and args.gpus != 1:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_desc(cfg, dtype):
    return (f"{cfg.name}: DCSBM N={cfg.n:,}, {cfg.blocks} blocks, E={cfg.edges:,} "
            f"(avg deg {2 * cfg.edges / cfg.n:.0f}), within:between {cfg.ratio:g}:1, "
            f"power-law degrees (exp -2.1, 10-100), k={cfg.k}, {dtype}")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index):
        self.dev = dev_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev_index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(cfg_n_local, nnz_local, n_global, k, es):
    """Compulsory bytes per launch of each hot kernel."""
    B = cfg_n_local * k * es
    return {
        # C2a: V once (every gathered row is a row of V), write AV, CSR + s
        "spmm": 2 * B + 4 * nnz_local + 8 * (cfg_n_local + 1) + 8 * n_global,
        # C2b: read V, X, AV
        "gram_stream": 3 * B,
        # C3: read X, V, AX, AV, Gp; write X, AX, G
        "update_direction": 8 * B,
        # C4: read G, Vp, X; write V
        "direction_gram": 4 * B,
    }


def iteration_bytes(n_local, nnz_local, n_global, k, es):
    """Algorithmic bytes of one whole iteration: 11 N x k block
    passes (X r/w, AX r/w, G r/w, V r/w, AV w/r, V read once by the SpMM) + the CSR
    pattern (4 nnz + 8 (N + 1)) + s (8 N)."""
    B = n_local * k * es
    return 11 * B + 4 * nnz_local + 8 * (n_local + 1) + 8 * n_global


def implementation_bytes(n_local, nnz_local, n_global, k, es):
    """Bytes this implementation's kernels must move at least (17 block passes:
    C3 8, C4 4, SpMM 2, C2b 3, + CSR + s); not the algorithmic figure."""
    B = n_local * k * es
    return 17 * B + 4 * nnz_local + 8 * (n_local + 1) + 8 * n_global


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def dmma_peak():
    """Measured fp64 tensor (DMMA.8x8x4) peak, TFLOP/s (profiles/r01/fp64_probe.txt)."""
    p = os.path.join(ROOT, "profiles", "r01", "fp64_probe.txt")
    try:
        for line in open(p):
            if line.startswith("DMMA tpb=256:"):
                return float(line.split(":")[1].split()[0]), "measured: tools/fp64_probe.cu (profiles/r01/fp64_probe.txt)"
    except OSError:
        pass
    return 40.0, "nominal B200 fp64 tensor (no measured file)"


def kernel_rooflines(kern, algo, n, k, method, hbm_peak, sm_mhz=None):
    """Per big kernel: average launch time, HBM fraction on its algorithmic bytes and
    fp64-tensor fraction on the algorithmic flops of its DMMA products (triu and the
    symmetric Grams count their upper triangle only); `binding` = the larger.  The DMMA
    peak was measured at the full 1965 MHz SM clock (64 FMA/clk/SM); with the run's
    median SM clock under load (`sm_mhz`, power capped) the same pipe peaks lower, which
    `fp64_tensor_frac_at_clock` reports beside the contract fraction."""
    tri = method.startswith("tri")
    f1 = method.endswith("f1")
    half = n * k * (k + 1)                     # one triangular / symmetric product
    full = 2 * n * k * k                       # one full N x k . k x k product
    flops = {
        "update_direction": (half if tri else full) * (1 if f1 else 2),
        "direction_gram": half + full,         # Q = V^T V (symmetric) + P = V^T X
        # T = V^T A V (symmetric) + R' = X^T A V; the f1 methods form only their
        # diagonals (k_gram_diag: 2 N k fp64 FMAs, no tensor products)
        "gram_stream": 0 if f1 else half + full,
        "spmm": 0,
    }
    tpk, tsrc = dmma_peak()
    out = {"fp64_tensor_peak_tflops": tpk, "fp64_tensor_peak_source": tsrc, "hbm_peak_gbs": hbm_peak}
    tpk_clk = tpk * sm_mhz / 1965.0 if sm_mhz else None
    if tpk_clk:
        out["fp64_tensor_peak_at_sm_clock_tflops"] = round(tpk_clk, 2)
        out["sm_mhz"] = sm_mhz
    for name in ("spmm", "update_direction", "direction_gram", "gram_stream"):
        if name not in kern or not kern[name]["launches"]:
            continue
        ms = kern[name]["ms_total"] / kern[name]["launches"]
        gbs = algo[name] / (ms / 1e3) / 1e9
        tf = flops[name] / (ms / 1e3) / 1e12
        fh, ft = gbs / hbm_peak, tf / tpk
        out[name] = {"avg_launch_ms": round(ms, 4), "hbm_gbs": round(gbs, 1), "hbm_frac": round(fh, 4),
                     "fp64_tensor_tflops": round(tf, 2), "fp64_tensor_frac": round(ft, 4),
                     "binding": "hbm" if fh >= ft else "fp64_tensor",
                     "algorithmic_bytes": algo[name], "algorithmic_flops": flops[name]}
        if tpk_clk:
            out[name]["fp64_tensor_frac_at_clock"] = round(tf / tpk_clk, 4)
    return out


def kp_of(k):
    return 16 if k <= 16 else 32 if k <= 32 else 48 if k <= 48 else 64


def nvlink_stats(info, kern, K, kp, es, world, max_over_ranks):
    """p > 1: halo exchange volume per rank per iteration (rows received / sent,
    DESIGN.md sec. 8) and the profiled (non-overlapped) communication time, as a
    fraction of 900 GB/s per direction per GPU (NVLink 5)."""
    if world == 1:
        return None
    recv_b = info["halo_rows"] * kp * es
    send_b = info["send_rows"] * kp * es
    comm_ms = kern.get("comm", {}).get("ms_total", 0.0) / max(K, 1)
    comm_ms = max_over_ranks(comm_ms)
    gbs = max(recv_b, send_b) / (comm_ms / 1e3) / 1e9 if comm_ms > 0 else None
    return {"halo_rows": info["halo_rows"], "send_rows": info["send_rows"],
            "recv_bytes_per_iter": recv_b, "send_bytes_per_iter": send_b,
            "allgather_bytes_per_iter": int((world - 1) * info["n"] / world * kp * es),
            "comm_ms_per_iter_profiled": round(comm_ms, 4),
            "achieved_gbs": round(gbs, 1) if gbs else None,
            "frac_of_900": round(gbs / 900.0, 4) if gbs else None,
            "allgather_probe": allgather_probe(info["n"], kp, es, world, max_over_ranks),
            "note": "profiled pass runs exchange and SpMM back to back; the timed pass overlaps "
                    "the exchange with the own-column part of the SpMM"}


def allgather_probe(n, kp, es, world, max_over_ranks, reps=5):
    """The achievable NVLink rate at the c4 message size: torch's
    all_gather_into_tensor of an (n / p) x KP block per rank, CUDA events, max over
    ranks; bus bandwidth = (p - 1) / p x total bytes / time, per GPU."""
    import torch
    import torch.distributed as dist
    rows = -(-n // world)
    elems = rows * kp
    dt = torch.float64 if es == 8 else torch.float32
    src = torch.ones(elems, dtype=dt, device="cuda")
    dst = torch.empty(elems * world, dtype=dt, device="cuda")
    dist.all_gather_into_tensor(dst, src)          # warm-up / connect
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    a.record()
    for _ in range(reps):
        dist.all_gather_into_tensor(dst, src)
    b.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / reps)
    total = elems * world * es
    busbw = (world - 1) / world * total / (ms / 1e3) / 1e9
    del src, dst
    torch.cuda.empty_cache()
    return {"bytes_per_rank_in": int(elems * (world - 1) * es), "ms": round(ms, 4),
            "bus_gbs": round(busbw, 1), "frac_of_900": round(busbw / 900.0, 4),
            "frac_of_measured_770": round(busbw / 770.0, 4)}


def load_gather_peak():
    """Measured L2-resident random-row gather bandwidth (tools/l2_bw_probe.cu)."""
    p = os.path.join(ROOT, "profiles", "measured_l2.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2305_10356_b200 as ofsc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = ofsc.Comm()
    cfg = CONFIGS[args.config]
    k = cfg.k
    es = 8 if args.dtype == "f64" else 4
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    t0 = time.time()
    src, dst, labels = config_graph(cfg)
    gen_s = time.time() - t0
    stream = torch.cuda.current_stream()

    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_a.record(stream)
    g = ofsc.Graph(cfg.n, src, dst, comm=comm, reorder=bool(args.reorder))
    ev_b.record(stream)
    torch.cuda.synchronize()
    build_ms = ev_a.elapsed_time(ev_b)
    info = g.info
    rb, re_ = info["row_begin"], info["row_end"]
    X0full = x0_block(cfg.n, k, cfg.seed_x0)
    if world == 1:
        X0 = X0full                                   # original order; the library permutes
    else:                                             # p > 1: this rank's internal rows
        X0 = X0full[g.copy_perm()[rb:re_]] if info["reordered"] else X0full[rb:re_]
    X0d = torch.from_numpy(X0).to(tdt).cuda()
    W, K = args.warmup, args.steps

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_run(method, profile=False):
        X = X0d.clone()
        barrier()
        r = ofsc.run(g, method, X, W + K, timing_skip=W, profile=profile, refresh=args.refresh)
        barrier()
        return r.report

    # --- headline: K timed iterations after W warm-up iterations, `passes` times
    # (median and minimum); value = the median pass ---
    clk = Clocks(local)
    pass_ms = []
    for _ in range(max(1, args.passes)):
        rep = timed_run(args.method)
        pass_ms.append(max_over_ranks(rep["timed_ms"]))
    clocks = clk.stop()
    ms = statistics.median(pass_ms)
    value = K / (ms / 1e3)

    # --- per-kernel profile pass (CUDA events per launch, same stream) ---
    prep = timed_run(args.method, profile=True)
    kern = {PHASES[i]: {"ms_total": prep["kernel_ms"][i], "launches": prep["kernel_launches"][i]}
            for i in range(10) if prep["kernel_launches"][i] or prep["kernel_ms"][i]}
    dom = max(("spmm", "update_direction", "direction_gram", "gram_stream"),
              key=lambda n: kern.get(n, {}).get("ms_total", 0.0))
    nl = re_ - rb
    algo = algorithmic_bytes(nl, info["nnz_local"], cfg.n, k, es)
    avg_ms = kern[dom]["ms_total"] / max(kern[dom]["launches"], 1)
    hbm_peak, peak_src = peaks()
    achieved = algo[dom] / (avg_ms / 1e3) / 1e9
    traffic = load_traffic()
    tr_bytes = None
    if traffic and traffic.get("config") == cfg.name and world == 1 and args.dtype == "f64":
        tr_bytes = (traffic.get("per_phase_dram_bytes") or {}).get(dom)
        if tr_bytes is None and traffic.get("kernel") == dom:
            tr_bytes = traffic.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "traffic": tr_bytes, "algorithmic_bytes_per_launch": algo[dom],
                "avg_launch_ms": round(avg_ms, 4), "peak_source": peak_src,
                "share_of_step": round(kern[dom]["ms_total"] / max(sum(v["ms_total"] for v in kern.values()), 1e-9), 3)}
    # The SpMM's neighbour-row gathers are served by L2/L1 (tools/l2_bw_probe.cu):
    # its second roofline is the measured L2 gather ceiling, with the bytes the
    # SMs must receive (one KP-wide row per stored nonzero + own row + output).
    gpk = load_gather_peak()
    kp = 16 if k <= 16 else 32 if k <= 32 else 48 if k <= 48 else 64
    gather_bytes = (info["nnz_local"] + 2 * nl) * kp * es
    sp_ms = kern["spmm"]["ms_total"] / max(kern["spmm"]["launches"], 1)
    roofline_l2 = None
    if gpk:
        ach = gather_bytes / (sp_ms / 1e3) / 1e9
        roofline_l2 = {"bound": "l2", "kernel": "spmm", "achieved": round(ach, 1),
                       "peak": gpk["l2_gather_gbs"], "unit": "GB/s",
                       "frac": round(ach / gpk["l2_gather_gbs"], 4),
                       "bytes_per_launch": gather_bytes, "avg_launch_ms": round(sp_ms, 4),
                       "peak_source": gpk["source"]}
    # every big kernel against both of its ceilings: HBM (algorithmic bytes, above)
    # and the fp64 tensor pipe (DMMA.8x8x4; algorithmic flops of its products)
    kr = kernel_rooflines(kern, algo, nl, k, args.method, hbm_peak, (clocks or {}).get("sm_mhz"))
    it_dram = None
    if traffic and traffic.get("config") == cfg.name and world == 1 and args.dtype == "f64" \
            and traffic.get("dram_bytes_per_iteration"):
        tb = traffic["dram_bytes_per_iteration"]
        it_dram = {"dram_bytes_per_iter": tb, "achieved_gbs": round(tb / (ms / K / 1e3) / 1e9, 1),
                   "frac": round(tb / (ms / K / 1e3) / 1e9 / hbm_peak, 4),
                   "source": traffic.get("source")}
    it_bytes = iteration_bytes(nl, info["nnz_local"], cfg.n, k, es)
    impl_bytes = implementation_bytes(nl, info["nnz_local"], cfg.n, k, es)

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "it/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic seeded DCSBM graph (stands in for the Graph Challenge SBM graphs, P:583-584)",
        "config": {"workload": workload_desc(cfg, args.dtype), "method": args.method, "k": k,
                   "refresh": args.refresh, "global_batch": cfg.n, "parallelism": f"row-partition p={world}",
                   "l2": "inputs larger than L2 (each N x k block 2.56 GB vs 126 MB L2)" if cfg.n * k * es > 2e8 else "working set partly L2-resident",
                   "graph_gen_s": round(gen_s, 1), "graph_build_ms": round(build_ms, 2),
                   "load_imbalance": info["load_imbalance"],
                   "reorder": ("LPA locality reordering derived from the graph (%d communities, "
                               "%.3f of nnz intra-community)" % (info["n_communities"],
                                                                  info["intra_edge_fraction"]))
                   if info["reordered"] else "none (random node ids)"},
        "roofline": roofline,
        "roofline_l2_gather": roofline_l2,
        "kernel_rooflines": kr,
        "iteration_dram_ncu": it_dram,
        "iteration_hbm": {"algorithmic_bytes_per_iter_per_gpu": it_bytes,
                          "definition": "11 B + 4 nnz + 8 (N + 1) + 8 N (SURVEY 8(d).3), B = N k w",
                          "achieved_gbs_per_gpu": round(it_bytes * (K / (ms / 1e3)) / 1e9, 1),
                          "frac": round(it_bytes * (K / (ms / 1e3)) / 1e9 / hbm_peak, 4),
                          "implementation_bytes_per_iter_per_gpu": impl_bytes,
                          "implementation_frac": round(impl_bytes * (K / (ms / 1e3)) / 1e9 / hbm_peak, 4)},
        "passes": {"n": len(pass_ms), "ms_per_step_median": round(ms / K, 4),
                   "ms_per_step_min": round(min(pass_ms) / K, 4),
                   "it_s_max": round(K / (min(pass_ms) / 1e3), 3),
                   "ms_per_step_all": [round(x / K, 4) for x in pass_ms]},
        "kernels": kern,
        "nvlink": nvlink_stats(info, kern, K, kp_of(k), es, world, max_over_ranks),
        "gpu_launches": rep["launches"],
        "clocks": clocks,
    }

    # --- Algorithm 1 stage breakdown on the resident graph (p == 1) ---
    if world == 1:
        def timed(fn):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            out_ = fn()
            b.record(stream)
            torch.cuda.synchronize()
            return out_, a.elapsed_time(b)
        X = X0d.clone()
        _, ms_run = timed(lambda: ofsc.run(g, args.method, X, cfg.iters, refresh=args.refresh))
        Y = torch.empty_like(X)
        _, ms_norm = timed(lambda: ofsc.row_normalize(X, Y))
        rows = torch.from_numpy(kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)).cuda()
        C0 = Y[rows].double().contiguous()
        (lab, km_it, _), ms_km = timed(lambda: ofsc.kmeans(Y, C0, 100))
        # NEXT-1: orthogonalisation + Rayleigh-Ritz + relerr on the features
        ofsc.rayleigh_ritz(g, X, want_vectors=False)      # warm-up (workspace, kernels)
        (theta, _, relerr), ms_rr = timed(lambda: ofsc.rayleigh_ritz(g, X, want_vectors=False))
        for _ in range(2):                 # second of two builds: warm allocation cache
            g0, ms_build_plain = timed(lambda: ofsc.Graph(cfg.n, src, dst, reorder=False))
            g0.close()
        for _ in range(2):
            g0, ms_build_warm = timed(lambda: ofsc.Graph(cfg.n, src, dst, reorder=bool(args.reorder)))
            g0.close()
        out["pipeline_ms"] = {
            "graph_build_first_in_process": round(build_ms, 2),
            "graph_build": round(ms_build_warm, 2), "graph_build_no_reorder": round(ms_build_plain, 2),
            f"run_{cfg.iters}_iters": round(ms_run, 2), "row_normalize": round(ms_norm, 3),
            "kmeans": round(ms_km, 2), "kmeans_lloyd_steps": km_it,
            "rayleigh_ritz": round(ms_rr, 2), "relerr": float(relerr),
            "ritz_values_min_max": [float(theta[0]), float(theta[-1])],
            "ari_vs_planted": round(ofsc.scores(lab.cpu().numpy(), labels)[0], 4)}

    # --- random node ids (no locality reordering): SURVEY 8(e) asks for this line ---
    if args.reorder and not args.no_random_ids:
        g.close()
        g_r = ofsc.Graph(cfg.n, src, dst, comm=comm, reorder=False)
        info_r = g_r.info
        X0r = X0full if world == 1 else X0full[info_r["row_begin"]:info_r["row_end"]]
        X0rd = torch.from_numpy(X0r).to(tdt).cuda()
        rms = []
        for _ in range(3):
            X = X0rd.clone()
            barrier()
            rr = ofsc.run(g_r, args.method, X, W + K, timing_skip=W, refresh=args.refresh)
            barrier()
            rms.append(max_over_ranks(rr.report["timed_ms"]))
        pr = ofsc.run(g_r, args.method, X0rd.clone(), W + K, timing_skip=W, profile=True,
                      refresh=args.refresh).report
        sp_r = pr["kernel_ms"][3] / max(pr["kernel_launches"][3], 1)
        out["random_ids"] = {
            "value": round(K / (statistics.median(rms) / 1e3), 3), "unit": "it/s",
            "ms_per_step": round(statistics.median(rms) / K, 4),
            "spmm_ms_per_launch": round(sp_r, 4),
            "load_imbalance": info_r["load_imbalance"],
            "what": "same workload, method and protocol on the graph with its random node ids "
                    "(no LPA reordering): the SpMM's neighbour gathers mostly miss L2"}
        del X0rd
        g_r.close()
        g = ofsc.Graph(cfg.n, src, dst, comm=comm, reorder=bool(args.reorder))

    # --- ARI / NMI vs planted blocks: mean over 10 k-means++ seeds ---
    if world == 1 and not args.no_ari:
        out["clustering"] = clustering_scores(ofsc, torch, g, args, cfg, X0d, labels)

    # --- all four methods, same protocol ---
    if not args.no_methods:
        per = {}
        for m in ofsc.METHODS:
            r = timed_run(m)
            per[m] = round(K / (max_over_ranks(r["timed_ms"]) / 1e3), 3)
        out["per_method_it_s"] = per
        # the f1 methods' C2b (k_gram_diag: diag T, diag R' only) against its ceiling
        if args.method.endswith("f2"):
            pf1 = timed_run("ofm_f1", profile=True)
            kf1 = {PHASES[i]: {"ms_total": pf1["kernel_ms"][i], "launches": pf1["kernel_launches"][i]}
                   for i in range(10) if pf1["kernel_launches"][i] or pf1["kernel_ms"][i]}
            out["kernel_rooflines_ofm_f1"] = kernel_rooflines(kf1, algo, nl, k, "ofm_f1", hbm_peak,
                                                              (clocks or {}).get("sm_mhz"))

    # --- e2e through the C ABI with pinned host buffers ---
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, cfg, comm, src, dst, X0full, world, rank, barrier, max_over_ranks)

    # --- CPU baseline: the oracle on the host cores (rank 0, N = 1 only) ---
    if world == 1 and rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(cfg, args.method, src, dst, X0full)

    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    g.close()
    if comm:
        comm.close()
        dist.destroy_process_group()


def kmeanspp_rows(torch, Y, K, seed):
    """k-means++ seeding (harness side): first row uniform, then rows
    drawn with probability proportional to the squared distance to the nearest
    chosen row.  Seeded (numpy PCG64), evaluated with torch on the device."""
    rng = np.random.default_rng(seed)
    n = Y.shape[0]
    rows = [int(rng.integers(n))]
    d2 = ((Y - Y[rows[0]]) ** 2).sum(1)
    for _ in range(1, K):
        cs = torch.cumsum(d2, 0)
        u = float(rng.random()) * float(cs[-1])
        i = int(torch.searchsorted(cs, torch.tensor([u], dtype=cs.dtype, device=cs.device)))
        i = min(i, n - 1)
        rows.append(i)
        d2 = torch.minimum(d2, ((Y - Y[i]) ** 2).sum(1))
    return rows


def clustering_scores(ofsc, torch, g, args, cfg, X0d, planted, seeds=10):
    """Algorithm 1 l.4-5 on the converged features (T = config iterations): row
    normalise, then K-means (K = planted blocks) from 10 k-means++ seeds; ARI and
    NMI against the planted blocks averaged over the seeds ("we repeat each
    experiment 10 times to record the average indexes")."""
    X = X0d.clone()
    ofsc.run(g, args.method, X, cfg.iters, refresh=args.refresh)
    Y = ofsc.row_normalize(X)
    Yd = Y.double()
    aris, nmis, inert = [], [], []
    for sd in range(seeds):
        rows = kmeanspp_rows(torch, Yd, cfg.blocks, cfg.seed_km + 1000 * sd)
        C0 = Yd[rows].contiguous()
        lab, it, inertia = ofsc.kmeans(Y, C0, 100)
        a, nm = ofsc.scores(lab.cpu().numpy(), planted)
        aris.append(a)
        nmis.append(nm)
        inert.append(inertia)
    return {"ari_mean": round(float(np.mean(aris)), 4), "ari_std": round(float(np.std(aris)), 4),
            "nmi_mean": round(float(np.mean(nmis)), 4), "nmi_std": round(float(np.std(nmis)), 4),
            "seeds": seeds, "iterations": cfg.iters, "init": "k-means++ (seeded, harness)",
            "inertia_min": float(min(inert)), "K": cfg.blocks}


def run_e2e(args, cfg, comm, src, dst, X0, world, rank, barrier, max_over_ranks):
    import ctypes as C
    import torch
    import paper_2305_10356_b200 as ofsc
    L = ofsc.lib()
    T = cfg.iters
    k = cfg.k
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    h_src = torch.from_numpy(src).pin_memory()
    h_dst = torch.from_numpy(dst).pin_memory()
    h_X0 = torch.from_numpy(X0).to(tdt).pin_memory()          # all n rows, original order
    h_X = torch.empty_like(h_X0).pin_memory()
    rows = torch.from_numpy(kmeans_init_rows(cfg.n, cfg.blocks, cfg.seed_km)).pin_memory()
    h_lab = torch.empty(cfg.n, dtype=torch.int32).pin_memory()
    o = ofsc.make_opts(k, T, refresh=args.refresh)
    stream = torch.cuda.current_stream()
    times = []
    for step in range(1 + args.e2e_steps):
        h_X.copy_(h_X0)                        # untimed host-side reset of the in/out buffer
        rep = ofsc.Report()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        st = L.ofsc_spectral_cluster(comm.handle if comm else None, cfg.n, src.size,
                                     C.c_void_p(h_src.data_ptr()), C.c_void_p(h_dst.data_ptr()),
                                     ofsc.METHODS[args.method], ofsc.DTYPES[args.dtype], C.byref(o),
                                     None, C.c_void_p(h_X.data_ptr()), cfg.blocks,
                                     C.c_void_p(rows.data_ptr()), 100,
                                     C.c_void_p(h_lab.data_ptr()), C.byref(rep),
                                     C.c_void_p(stream.cuda_stream))
        b.record(stream)
        barrier()
        ofsc._check(st)
        if step >= 1:
            times.append(max_over_ranks(a.elapsed_time(b)))
    ms = statistics.median(times)       # median of the timed calls (first-call outliers)
    ari, nmi = (None, None)
    if world == 1:
        ari, nmi = ofsc.scores(h_lab.numpy(), config_graph(cfg)[2])
    es = 8 if args.dtype == "f64" else 4
    h2d = src.nbytes + dst.nbytes + X0.shape[0] * k * es + rows.numel() * 8
    d2h = X0.shape[0] * k * es + cfg.n * 4
    return {"value": round(T / (ms / 1e3), 3), "unit": "it/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "bytes_counted_per": f"call (one ofsc_spectral_cluster = {T} iterations + build + K-means)",
            "h2d_bytes_per_iteration": int(h2d // T), "d2h_bytes_per_iteration": int(d2h // T),
            "ms_per_call": round(ms, 2), "ms_per_call_is": "median of the timed calls",
            "iters_per_call": T,
            "calls_timed": len(times), "ms_calls": [round(t, 1) for t in times],
            "what": "ofsc_spectral_cluster: edge H2D + GPU CSR build + T iterations + row "
                    "normalise + K-means (K = planted blocks, <= 100 Lloyd steps) + D2H",
            "ari_vs_planted": ari, "nmi_vs_planted": nmi}


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(th) if th else 1
    except Exception:
        return 1


class OracleSampler:
    """Bounded samples of the oracle's iteration (oracle/sample.py): one sample =
    Algorithm 2's arithmetic on a block of ~N/blocks rows, timed and scaled by
    N / rows to a full-iteration rate.  Setup (operator build, the first A X and
    direction over all rows) is untimed."""

    def __init__(self, cfg, method, src, dst, X0):
        from oracle import build_operator, apply_A, direction
        self.method = method
        self.op = build_operator(cfg.n, src, dst)
        self.X = np.asarray(X0, dtype=np.float64)
        self.AX = apply_A(self.op, self.X)
        self.M = self.X.T @ self.X
        self.W = self.X.T @ self.AX
        self.Gp = direction(method, self.X, self.AX, self.M, self.W)
        self.Vp = -self.Gp
        from oracle import colsum
        self.gg_prev = colsum(self.Gp * self.Gp)      # PR denominator over all rows
        n = cfg.n
        self.blocks = 1 if n <= 250_000 else max(1, int(round(n / 312_500)))   # ~1-2 s per sample at c4
        self.bounds = np.linspace(0, n, self.blocks + 1).astype(np.int64)
        self.n = n
        self.i = 0
        # untimed views: the row slices of S (a copy in scipy) and s * Vp (each
        # sample recomputes its own rows' share of it)
        self.S_rows = [self.op.S[int(self.bounds[b]):int(self.bounds[b + 1])] for b in range(self.blocks)]
        self.sVp = self.op.s[:, None] * self.Vp

    def step(self):
        """Run one sample; return (seconds, rows)."""
        from oracle.sample import iteration_rows
        b = self.i % self.blocks
        self.i += 1
        r0, r1 = int(self.bounds[b]), int(self.bounds[b + 1])
        t = time.perf_counter()
        iteration_rows(self.op, self.method, self.X, self.AX, self.Gp, self.Vp, self.M, self.W,
                       r0, r1, S_rows=self.S_rows[b], sVp=self.sVp, gg_prev=self.gg_prev)
        return time.perf_counter() - t, r1 - r0

    def describe(self, cfg, nsteps):
        return (f"{nsteps} samples of one {self.method} iteration of {cfg.name}, each on a block of "
                f"~{self.n // self.blocks:,} of the {self.n:,} rows (Algorithm 2's arithmetic: direction, "
                f"SpMM rows, Grams, k x k line search, update; oracle/sample.py); value = rows processed "
                f"/ N per second; scipy SpMM single-threaded, numpy BLAS with {oracle_threads()} threads")


def cpu_baseline(cfg, method, src, dst, X0, iters=2):
    """The oracle as it stands (oracle.run_ofm, Algorithm 2, numpy + scipy) on the host
    cores: `iters` WHOLE iterations of the workload (c4, 2
    iterations), timed between the oracle's own per-iteration callbacks after one
    untimed iteration (operator build and the first iteration excluded)."""
    from oracle import build_operator, run_ofm
    op = build_operator(cfg.n, src, dst)
    stamps = []
    run_ofm(op, method, X0, iters + 1, refresh=0,
            callback=lambda t: stamps.append(time.perf_counter()))
    secs = stamps[-1] - stamps[0]
    return {"value": round(iters / secs, 5), "unit": "it/s", "cores": oracle_threads(),
            "kind": "oracle", "host_cpus": os.cpu_count(),
            "sample": f"{iters} whole {method} iterations of {cfg.name} (all {cfg.n:,} rows; "
                      f"oracle.run_ofm, refresh = 0 as the GPU run) after one untimed iteration: "
                      f"{secs:.1f} s; scipy SpMM single-threaded, numpy BLAS with "
                      f"{oracle_threads()} threads"}


# ---------------------------------------------------------------------------
def run_reference(args):
    """Reference arm: the oracle, as it stands, on this box's host cores (rank 0 only).
    Each step is a bounded sample of the workload (OracleSampler): one iteration's
    arithmetic on a block of ~N/16 rows.  ms_per_step is the measured time of one
    sample; value = (iterations' worth of rows processed) / (time), in it/s."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    if world > 1:
        # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 alone runs the oracle
        # here, so give its BLAS the host cores it has at N = 1 (same oracle, same threads)
        try:
            from threadpoolctl import threadpool_limits
            threadpool_limits(len(os.sched_getaffinity(0)))
        except Exception:
            pass
    cfg = CONFIGS[args.config]
    src, dst, _ = config_graph(cfg)
    X0 = x0_block(cfg.n, cfg.k, cfg.seed_x0)
    smp = OracleSampler(cfg, args.method, src, dst, X0)
    W, K = args.warmup, args.steps
    for _ in range(W):
        smp.step()
    secs = rows = 0.0
    for _ in range(K):
        dt, r = smp.step()
        secs += dt
        rows += r
    per_iter = secs * cfg.n / rows
    value = 1.0 / per_iter
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "it/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(1e3 * secs / K, 2),
        "step_is": f"one bounded sample = {rows / K / cfg.n:.4f} of an iteration (rows block)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic seeded DCSBM graph", "config": {"workload": workload_desc(cfg, "f64"),
                                                         "method": args.method, "k": cfg.k},
        "cpu_baseline": {"value": round(value, 5), "unit": "it/s", "cores": oracle_threads(),
                         "kind": "oracle", "sample": smp.describe(cfg, K)},
        "e2e": {"value": round(value, 5), "unit": "it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    a = parse()
    launch_ranks(a)
    if a.dry_run:
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")),
                          "world": int(os.environ.get("WORLD_SIZE", "1")),
                          "gpus": a.gpus}), flush=True)
        sys.exit(0)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)

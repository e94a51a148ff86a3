"""Summarise tools/ncu_iter.sh output: per-kernel metrics of the last full
iteration (c4) -> profiles/<round>/ncu_iter_summary.json and the per-kernel DRAM
bytes that bench.py reads (profiles/ncu_traffic.json)."""
import csv
import json
import os
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_iter/iter_metrics.csv"
dst_dir = sys.argv[2] if len(sys.argv) > 2 else "profiles/r01"
rows = [r for r in csv.reader(open(src)) if r and r[0].isdigit()]
hdr = None
for r in csv.reader(open(src)):
    if r and r[0] == "ID":
        hdr = r
        break
ix = {n: i for i, n in enumerate(hdr)}
launch = {}
for r in rows:
    lid = int(r[ix["ID"]])
    d = launch.setdefault(lid, {"kernel": r[ix["Kernel Name"]]})
    val = r[ix["Metric Value"]].replace(",", "")
    unit = r[ix["Metric Unit"]]
    try:
        v = float(val)
    except ValueError:
        continue
    if unit == "byte":
        v = v
    elif unit == "Kbyte":
        v *= 1e3
    elif unit == "Mbyte":
        v *= 1e6
    elif unit == "Gbyte":
        v *= 1e9
    elif unit in ("nsecond", "ns"):
        v *= 1e-6
    elif unit in ("usecond", "us"):
        v *= 1e-3
    elif unit in ("msecond", "ms"):
        v *= 1.0
    elif unit == "second":
        v *= 1e3
    d[r[ix["Metric Name"]]] = v
ids = sorted(launch)
short = {"k_update_direction": "update_direction", "k_direction_gram": "direction_gram",
         "k_spmm": "spmm", "k_gram_stream": "gram_stream", "k_gram_diag": "gram_stream",
         "k_beta": "beta",
         "k_linesearch": "line_search", "k_reduce_linesearch": "line_search",
         "k_reduce_partials": "gram_reduce"}
# the last iteration: the last k_update_direction launch and what follows it
last_c3 = max(i for i in ids if launch[i]["kernel"].startswith("void ofsc::k_update_direction")
              or launch[i]["kernel"].startswith("k_update_direction"))
it = []
for i in ids:                                   # one iteration: C3 ... line search
    if i < last_c3:
        continue
    it.append(launch[i])
    if "linesearch" in launch[i]["kernel"]:       # k_linesearch or k_reduce_linesearch
        break
summ = []
for d in it:
    name = d["kernel"].replace("void ", "").replace("ofsc::", "").split("(")[0]
    base = name.split("<")[0]
    e = {"kernel": name, "phase": short.get(base, base)}
    for k, v in d.items():
        if k != "kernel":
            e[k] = round(v, 4) if isinstance(v, float) else v
    summ.append(e)
os.makedirs(dst_dir, exist_ok=True)
json.dump(summ, open(os.path.join(dst_dir, "ncu_iter_summary.json"), "w"), indent=1)
per = {}
tot_bytes = 0.0
tot_ms = 0.0
for e in summ:
    b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    per.setdefault(e["phase"], 0.0)
    per[e["phase"]] += b
    tot_bytes += b
    tot_ms += e.get("gpu__time_duration.sum", 0)
traffic = {"config": "c4", "kernel": "spmm", "dram_bytes_per_launch": per.get("spmm"),
           "dram_bytes_per_iteration": tot_bytes, "per_phase_dram_bytes": per,
           "ncu_iteration_ms": tot_ms,
           "source": f"{dst_dir}/ncu_iter_summary.json (ncu --clock-control none, c4 reordered, OFM-f2, last iteration of tools/run_iters.py)"}
if "notraffic" not in sys.argv[3:]:      # the bench's traffic figure is the OFM-f2 run's
    json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
for e in summ:
    print(f"{e['kernel'][:40]:40s} {e.get('gpu__time_duration.sum', 0):8.3f} ms  "
          f"DRAM {(e.get('dram__bytes_read.sum', 0) + e.get('dram__bytes_write.sum', 0)) / 1e9:7.2f} GB  "
          f"tensor {e.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
          f"L1 {e.get('l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%  "
          f"L2 {e.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")
print("iteration DRAM GB", tot_bytes / 1e9, "ncu ms", tot_ms)

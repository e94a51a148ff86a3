"""Build libofsc.so in-tree (nvcc, sm_100a only).

Usage: python -m paper_2305_10356_b200._build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ofsc")
LIB = os.path.join(PKG, "libofsc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# translation units whose scalar arithmetic must round exactly as written
NO_FMAD = {"kernels_ls.cu", "kernels_kmeans.cu"}


def nccl_dirs():
    """The NCCL that torch loads (pip wheel), so one libnccl.so.2 is in the process."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        inc, lib = os.path.join(c, "include"), os.path.join(c, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("NCCL headers not found")


def _compile(src, obj, inc):
    flags = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    if os.path.basename(src) in NO_FMAD:
        flags.append("-fmad=false")
    cmd = flags + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = obj + ".log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "ofsc.h"), __file__]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s in srcs:
            obj = os.path.join(BUILD, os.path.basename(s) + ".o")
            if force or not os.path.exists(obj) or os.path.getmtime(obj) < newest:
                jobs.append(ex.submit(_compile, s, obj, inc))
        for j in jobs:
            o = j.result()
            if verbose:
                print("compiled", os.path.basename(o), flush=True)
    objs = [os.path.join(BUILD, os.path.basename(s) + ".o") for s in srcs]
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("linked", LIB, flush=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)

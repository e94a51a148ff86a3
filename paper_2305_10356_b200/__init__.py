"""paper_2305_10356_b200 -- orthogonalization-free spectral clustering on B200.

Thin ctypes binding of libofsc.so (include/ofsc.h).  Argument marshalling
only: every numerical step runs in the library's sm_100a kernels.  There is no
CPU fallback; importing works without a GPU (so the ABI can be inspected), but
every compute call needs the CUDA device and the in-tree libofsc.so, and fails
loudly otherwise.

Names follow the paper (arXiv 2305.10356): methods OFM-f1, TriOFM-f1, OFM-f2,
TriOFM-f2, Algorithm 1, Algorithm 2.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libofsc.so")

METHODS = {"ofm_f1": 0, "triofm_f1": 1, "ofm_f2": 2, "triofm_f2": 3}
DTYPES = {"f64": 0, "f32": 1}
BETA_RULES = {"pr": 0, "pr+": 1, "zero": 2}
MAX_K = 64


class OfscError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"ofsc status {status}: {msg}")
        self.status = status


class OfscDiverged(OfscError):
    pass


class Opts(C.Structure):
    _fields_ = [("k", C.c_int32), ("max_iters", C.c_int32), ("tol", C.c_double),
                ("beta_rule", C.c_int32), ("line_search", C.c_int32),
                ("alpha_fixed", C.c_double), ("refresh", C.c_int32),
                ("check_every", C.c_int32), ("timing_skip", C.c_int32), ("profile", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("diverged", C.c_int32),
                ("n_three_root_steps", C.c_int32), ("n_zero_steps", C.c_int32),
                ("grad_norm0", C.c_double), ("grad_norm", C.c_double),
                ("objective", C.c_double), ("timed_iters", C.c_int32), ("launches", C.c_int32),
                ("timed_ms", C.c_double), ("kernel_ms", C.c_double * 10),
                ("kernel_launches", C.c_int32 * 10)]

    def as_dict(self):
        out = {}
        for f, _ in self._fields_:
            v = getattr(self, f)
            out[f] = list(v) if f in ("kernel_ms", "kernel_launches") else v
        return out


class GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_edges_kept", C.c_int64), ("nnz_global", C.c_int64),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("nnz_local", C.c_int64),
                ("n_isolated", C.c_int64), ("n_self_loops_dropped", C.c_int64),
                ("n_duplicates_dropped", C.c_int64), ("max_degree", C.c_int64),
                ("fro2_A", C.c_double), ("load_imbalance", C.c_double),
                ("reordered", C.c_int32), ("n_communities", C.c_int64),
                ("intra_edge_fraction", C.c_double), ("halo_rows", C.c_int64),
                ("send_rows", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class BuildOpts(C.Structure):
    _fields_ = [("reorder", C.c_int32), ("lpa_sweeps", C.c_int32)]


# exported symbol -> (restype, argtypes); mirrors include/ofsc.h
_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_ST = C.c_int
SIGNATURES = {
    "ofsc_version": (C.c_char_p, []),
    "ofsc_trim_memory": (_ST, []),
    "ofsc_status_string": (C.c_char_p, [_ST]),
    "ofsc_last_error": (C.c_char_p, []),
    "ofsc_get_unique_id": (_ST, [_P]),
    "ofsc_comm_create": (_ST, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "ofsc_comm_destroy": (_ST, [_P]),
    "ofsc_comm_create_local": (_ST, [C.c_int, C.c_int, C.POINTER(_P)]),
    "ofsc_comm_create_local_world": (_ST, [C.c_int, C.POINTER(_P)]),
    "ofsc_partition_rows": (_ST, [_I64, _P, C.c_int, _P]),
    "ofsc_graph_build": (_ST, [_P, _I64, _I64, _P, _P, C.c_int, _P, C.POINTER(_P)]),
    "ofsc_graph_build_ex": (_ST, [_P, _I64, _I64, _P, _P, C.c_int, C.POINTER(BuildOpts), _P,
                                  C.POINTER(_P)]),
    "ofsc_graph_info_get": (_ST, [_P, C.POINTER(GraphInfo)]),
    "ofsc_graph_append": (_ST, [_P, _I64, _P, _P, C.c_int, _P]),
    "ofsc_graph_exchange_plan": (_ST, [_P, _P, _P, _P, _P]),
    "ofsc_graph_copy_csr": (_ST, [_P, _P, _P, _P]),
    "ofsc_graph_copy_perm": (_ST, [_P, _P]),
    "ofsc_graph_destroy": (_ST, [_P]),
    "ofsc_graph_apply": (_ST, [_P, _ST, _I32, _P, _I64, _P, _I64, _P]),
    "ofsc_graph_apply_gram": (_ST, [_P, _ST, _I32, _P, _I64, _P, _I64, _P, _I64, _P, _P]),
    "ofsc_opts_default": (None, [C.POINTER(Opts)]),
    "ofsc_run": (_ST, [_P, _ST, _ST, C.POINTER(Opts), _P, _I64, _P, C.POINTER(Report), _P]),
    "ofsc_run_ex": (_ST, [_P, _ST, _ST, C.POINTER(Opts), _P, _I64, _P, _P, _P,
                          C.POINTER(Report), _P]),
    "ofsc_line_search": (_ST, [_ST, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ofsc_row_normalize": (_ST, [_ST, _I64, _I32, _P, _I64, _P, _I64, _P]),
    "ofsc_kmeans": (_ST, [_P, _ST, _I64, _I32, _P, _I64, _I32, _P, _I32, _P, _P, _P, _P]),
    "ofsc_scores": (_ST, [_I64, _P, _P, _P, _P]),
    "ofsc_rayleigh_ritz": (_ST, [_P, _ST, _I32, _P, _I64, _P, _I64, _P, _P, _P]),
    "ofsc_spectral_cluster": (_ST, [_P, _I64, _I64, _P, _P, _ST, _ST, C.POINTER(Opts),
                                    C.POINTER(BuildOpts), _P, _I32, _P, _I32, _P,
                                    C.POINTER(Report), _P]),
}

_lib = None


def lib():
    """Load libofsc.so (in-tree).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "(python -m paper_2305_10356_b200._build)")
        try:
            import torch  # noqa: F401  (load torch's libnccl/cudart first: one NCCL per process)
        except Exception:
            pass
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        msg = lib().ofsc_last_error().decode()
        if st == 6:
            raise OfscDiverged(st, msg)
        raise OfscError(st, msg)


def version():
    return lib().ofsc_version().decode()


def trim_memory():
    """Release the library's cached device blocks and trim its pool (ofsc_trim_memory)."""
    _check(lib().ofsc_trim_memory())


# ---------------------------------------------------------------------------
# torch marshalling helpers
# ---------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dt_of(t):
    torch = _torch()
    if t.dtype == torch.float64:
        return 0
    if t.dtype == torch.float32:
        return 1
    raise TypeError("features must be float64 or float32")


def _dev2d(t):
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dim() == 2 and t.stride(1) == 1):
        raise TypeError("expected a 2-D CUDA tensor with unit column stride")
    return t


class Comm:
    """NCCL communicator over torch.distributed ranks (one process per GPU)."""

    @staticmethod
    def broadcast_unique_id(group=None) -> bytes:
        """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
        import torch.distributed as dist
        torch = _torch()
        uid = torch.zeros(128, dtype=torch.uint8)
        if dist.get_rank(group) == 0:
            buf = (C.c_ubyte * 128)()
            _check(lib().ofsc_get_unique_id(C.cast(buf, C.c_void_p)))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            uid = uid.cuda()
        dist.broadcast(uid, 0, group=group)
        return bytes(uid.cpu().tolist())

    def __init__(self, group=None):
        import torch.distributed as dist
        torch = _torch()
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        raw = Comm.broadcast_unique_id(group)
        buf = (C.c_ubyte * 128).from_buffer_copy(raw)
        h = C.c_void_p()
        _check(lib().ofsc_comm_create(C.cast(buf, C.c_void_p), self.size, self.rank,
                                      torch.cuda.current_device(), C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            _check(lib().ofsc_comm_destroy(self.handle))
            self.handle = None


class LocalComm:
    """Test communicator (no NCCL): rank `rank` of `size` in this process (see
    ofsc_comm_create_local).  Graph build and kernel hooks only."""

    def __init__(self, size, rank):
        h = C.c_void_p()
        _check(lib().ofsc_comm_create_local(int(size), int(rank), C.byref(h)))
        self.handle, self.size, self.rank = h, size, rank

    def close(self):
        if self.handle:
            _check(lib().ofsc_comm_destroy(self.handle))
            self.handle = None


class LocalWorld:
    """In-process world of `size` ranks on the current GPU without NCCL
    (ofsc_comm_create_local_world): every call runs the full p > 1 schedule
    (halo exchange, rank-order sums, split SpMM) between the ranks.  Each rank
    must be driven by its own host thread: use `run`."""

    class _RankComm:
        def __init__(self, handle, size, rank):
            self.handle, self.size, self.rank = handle, size, rank

        def close(self):
            if self.handle:
                _check(lib().ofsc_comm_destroy(self.handle))
                self.handle = None

    def __init__(self, size):
        arr = (C.c_void_p * int(size))()
        _check(lib().ofsc_comm_create_local_world(int(size), arr))
        self.size = int(size)
        self.comms = [LocalWorld._RankComm(C.c_void_p(arr[r]), self.size, r)
                      for r in range(self.size)]

    def run(self, fn, timeout=900.0):
        """fn(rank, comm) on one host thread per rank (each with its own CUDA stream);
        returns the per-rank results, re-raising the first exception.  A rank that
        fails outside a collective leaves the others waiting at the next one: the
        threads are daemons and `timeout` (s) turns that into a TimeoutError."""
        import threading
        torch = _torch()
        dev = torch.cuda.current_device()
        out = [None] * self.size
        err = [None] * self.size

        def body(r):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(torch.cuda.Stream()):
                    out[r] = fn(r, self.comms[r])
                    torch.cuda.current_stream().synchronize()
            except BaseException as e:  # noqa: BLE001 (re-raised below)
                err[r] = e

        ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.size)]
        for t in ths:
            t.start()
        for t in ths:
            t.join(timeout)
        for e in err:
            if e is not None:
                raise e
        if any(t.is_alive() for t in ths):
            raise TimeoutError("local world: a rank did not reach a collective")
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        for c in self.comms:
            c.close()


def partition_rows(row_ptr, p):
    """nnz-balanced contiguous row split (host function of the library)."""
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
    out = np.empty(int(p) + 1, np.int64)
    _check(lib().ofsc_partition_rows(rp.size - 1, rp.ctypes.data_as(C.c_void_p), int(p),
                                     out.ctypes.data_as(C.c_void_p)))
    return out


class Graph:
    """Shifted normalised Laplacian A = L - 2I of an undirected graph."""

    def __init__(self, n, src, dst, comm: Comm | None = None, stream=None, reorder=False,
                 lpa_sweeps=30):
        torch = _torch()
        self.n = int(n)
        self.comm = comm
        h = C.c_void_p()
        bo = BuildOpts(1 if reorder else 0, int(lpa_sweeps))
        if isinstance(src, torch.Tensor) and src.is_cuda:
            s = src.to(torch.int64).contiguous()
            d = dst.to(torch.int64).contiguous()
            _check(lib().ofsc_graph_build_ex(comm.handle if comm else None, self.n, s.numel(),
                                             C.c_void_p(s.data_ptr()), C.c_void_p(d.data_ptr()),
                                             1, C.byref(bo), _stream(stream), C.byref(h)))
        else:
            s = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
            d = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
            _check(lib().ofsc_graph_build_ex(comm.handle if comm else None, self.n, s.size,
                                             s.ctypes.data_as(C.c_void_p),
                                             d.ctypes.data_as(C.c_void_p), 0, C.byref(bo),
                                             _stream(stream), C.byref(h)))
        self.handle = h
        self.info = self.get_info()

    def append(self, src, dst, stream=None):
        """Add a batch of edges in place (ofsc_graph_append; streaming snapshots)."""
        torch = _torch()
        if isinstance(src, torch.Tensor) and src.is_cuda:
            s = src.to(torch.int64).contiguous()
            d = dst.to(torch.int64).contiguous()
            _check(lib().ofsc_graph_append(self.handle, s.numel(), C.c_void_p(s.data_ptr()),
                                           C.c_void_p(d.data_ptr()), 1, _stream(stream)))
        else:
            s = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
            d = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
            _check(lib().ofsc_graph_append(self.handle, s.size, s.ctypes.data_as(C.c_void_p),
                                           d.ctypes.data_as(C.c_void_p), 0, _stream(stream)))
        self.info = self.get_info()

    def exchange_plan(self):
        """(send_counts[p], send_gids, recv_counts[p], recv_gids) of this rank (p > 1)."""
        p = self.comm.size if self.comm is not None else 1
        sc = np.zeros(p, np.int64)
        rc = np.zeros(p, np.int64)
        sg = np.zeros(max(self.info["send_rows"], 1), np.int32)
        rg = np.zeros(max(self.info["halo_rows"], 1), np.int32)
        _check(lib().ofsc_graph_exchange_plan(self.handle, sc.ctypes.data_as(C.c_void_p),
                                              sg.ctypes.data_as(C.c_void_p),
                                              rc.ctypes.data_as(C.c_void_p),
                                              rg.ctypes.data_as(C.c_void_p)))
        return sc, sg[:self.info["send_rows"]], rc, rg[:self.info["halo_rows"]]

    def get_info(self):
        gi = GraphInfo()
        _check(lib().ofsc_graph_info_get(self.handle, C.byref(gi)))
        return gi.as_dict()

    @property
    def n_local(self):
        return self.info["row_end"] - self.info["row_begin"]

    def copy_csr(self):
        nl = self.n_local
        rp = np.empty(nl + 1, np.int64)
        col = np.empty(max(self.info["nnz_local"], 1), np.int32)
        s = np.empty(self.n, np.float64)
        _check(lib().ofsc_graph_copy_csr(self.handle, rp.ctypes.data_as(C.c_void_p),
                                         col.ctypes.data_as(C.c_void_p),
                                         s.ctypes.data_as(C.c_void_p)))
        return rp, col[:self.info["nnz_local"]], s

    def copy_perm(self):
        """perm[i] = original node id of internal row i (identity unless reordered)."""
        perm = np.empty(self.n, np.int32)
        _check(lib().ofsc_graph_copy_perm(self.handle, perm.ctypes.data_as(C.c_void_p)))
        return perm

    def apply(self, Z, Y=None, stream=None):
        """Y = A Z for the local rows (Z holds all n rows)."""
        torch = _torch()
        Z = _dev2d(Z)
        k = Z.shape[1]
        if Y is None:
            Y = torch.empty((self.n_local, k), dtype=Z.dtype, device=Z.device)
        _check(lib().ofsc_graph_apply(self.handle, _dt_of(Z), k, C.c_void_p(Z.data_ptr()),
                                      Z.stride(0), C.c_void_p(Y.data_ptr()), Y.stride(0),
                                      _stream(stream)))
        return Y

    def apply_gram(self, Z, X, stream=None):
        """SpMM + Gram hook (C2a then C2b): Y = A Z and (Z^T Z, Z^T X, Z^T Y, X^T Y)."""
        torch = _torch()
        Z, X = _dev2d(Z), _dev2d(X)
        k = Z.shape[1]
        Y = torch.empty((self.n_local, k), dtype=Z.dtype, device=Z.device)
        G = torch.empty((4, k, k), dtype=torch.float64, device=Z.device)
        _check(lib().ofsc_graph_apply_gram(self.handle, _dt_of(Z), k, C.c_void_p(Z.data_ptr()),
                                           Z.stride(0), C.c_void_p(X.data_ptr()), X.stride(0),
                                           C.c_void_p(Y.data_ptr()), Y.stride(0),
                                           C.c_void_p(G.data_ptr()), _stream(stream)))
        return Y, G

    def close(self):
        if getattr(self, "handle", None):
            lib().ofsc_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PHASES = ("update_direction", "beta", "direction_gram", "spmm", "gram_reduce",
          "line_search", "refresh", "comm", "gram_stream", "unused")


def make_opts(k, max_iters, tol=0.0, beta_rule="pr+", line_search=True, alpha_fixed=0.0,
              refresh=0, check_every=8, timing_skip=-1, profile=False):
    o = Opts()
    lib().ofsc_opts_default(C.byref(o))
    o.k, o.max_iters, o.tol = int(k), int(max_iters), float(tol)
    o.beta_rule = BETA_RULES[beta_rule]
    o.line_search = 1 if line_search else 0
    o.alpha_fixed = float(alpha_fixed)
    o.refresh = int(refresh)
    o.check_every = int(check_every)
    o.timing_skip = int(timing_skip)
    o.profile = 1 if profile else 0
    return o


@dataclass
class RunResult:
    report: dict
    history: np.ndarray
    alphas: np.ndarray | None = None
    codes: np.ndarray | None = None


def run(graph: Graph, method: str, X, max_iters, *, tol=0.0, beta_rule="pr+",
        line_search=True, alpha_fixed=0.0, refresh=0, check_every=8, debug=False,
        timing_skip=-1, profile=False, raise_on_diverge=True, stream=None) -> RunResult:
    """Algorithm 2 on the device; X (local rows x k CUDA tensor) is updated in place."""
    X = _dev2d(X)
    k = X.shape[1]
    o = make_opts(k, max_iters, tol, beta_rule, line_search, alpha_fixed, refresh, check_every,
                  timing_skip, profile)
    T = int(max_iters)
    hist = np.full((max(T, 1), 4), np.nan)
    rep = Report()
    al = np.empty((max(T, 1), k)) if debug else None
    cd = np.empty((max(T, 1), k), np.int32) if debug else None
    st = lib().ofsc_run_ex(graph.handle, METHODS[method], _dt_of(X), C.byref(o),
                           C.c_void_p(X.data_ptr()), X.stride(0), hist.ctypes.data_as(C.c_void_p),
                           al.ctypes.data_as(C.c_void_p) if debug else None,
                           cd.ctypes.data_as(C.c_void_p) if debug else None,
                           C.byref(rep), _stream(stream))
    if st == 6 and not raise_on_diverge:
        pass
    else:
        _check(st)
    return RunResult(rep.as_dict(), hist[:T], al[:T] if debug else None,
                     cd[:T] if debug else None)


def line_search(method, Q, P, T, Rp, M, W):
    """k x k exact line search on the device from host Grams (kernel-level hook)."""
    k = Q.shape[0]
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (Q, P, T, Rp, M, W)]
    alpha = np.empty(k)
    codes = np.empty(k, np.int32)
    Mo = np.empty((k, k))
    Wo = np.empty((k, k))
    _check(lib().ofsc_line_search(METHODS[method], k,
                                  *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                  alpha.ctypes.data_as(C.c_void_p), codes.ctypes.data_as(C.c_void_p),
                                  Mo.ctypes.data_as(C.c_void_p), Wo.ctypes.data_as(C.c_void_p)))
    return alpha, codes, Mo, Wo


def row_normalize(X, Y=None, stream=None):
    torch = _torch()
    X = _dev2d(X)
    if Y is None:
        Y = torch.empty_like(X)
    _check(lib().ofsc_row_normalize(_dt_of(X), X.shape[0], X.shape[1], C.c_void_p(X.data_ptr()),
                                    X.stride(0), C.c_void_p(Y.data_ptr()), Y.stride(0),
                                    _stream(stream)))
    return Y


def kmeans(Y, centroids, max_iters=100, comm: Comm | None = None, stream=None):
    """Lloyd K-means from the given centroids (K x dim float64 CUDA tensor, updated in place)."""
    torch = _torch()
    Y = _dev2d(Y)
    assert centroids.dtype == torch.float64 and centroids.is_cuda and centroids.is_contiguous()
    labels = torch.empty(Y.shape[0], dtype=torch.int32, device=Y.device)
    it = C.c_int32()
    inertia = C.c_double()
    _check(lib().ofsc_kmeans(comm.handle if comm else None, _dt_of(Y), Y.shape[0], Y.shape[1],
                             C.c_void_p(Y.data_ptr()), Y.stride(0), centroids.shape[0],
                             C.c_void_p(centroids.data_ptr()), int(max_iters),
                             C.c_void_p(labels.data_ptr()), C.byref(it), C.byref(inertia),
                             _stream(stream)))
    return labels, it.value, inertia.value


def rayleigh_ritz(graph, X, want_vectors=True, stream=None):
    """Orthogonalisation + Rayleigh-Ritz on span(X) and relerr (ofsc_rayleigh_ritz;
    P:589).  X: local rows x k CUDA tensor (fp64 or fp32), not modified.
    Returns (theta float64[k] ascending (numpy), U (same shape/dtype as X) or None, relerr)."""
    torch = _torch()
    X = _dev2d(X)
    k = X.shape[1]
    U = torch.empty_like(X) if want_vectors else None
    theta = np.zeros(k, dtype=np.float64)
    rel = C.c_double()
    _check(lib().ofsc_rayleigh_ritz(graph.handle, _dt_of(X), k, C.c_void_p(X.data_ptr()),
                                    X.stride(0), C.c_void_p(U.data_ptr()) if U is not None else None,
                                    U.stride(0) if U is not None else k,
                                    theta.ctypes.data_as(C.c_void_p), C.byref(rel),
                                    _stream(stream)))
    return theta, U, rel.value


def scores(a, b):
    """(ARI, NMI) of two labelings (host)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.int32))
    ari, nmi = C.c_double(), C.c_double()
    _check(lib().ofsc_scores(a.size, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                             C.byref(ari), C.byref(nmi)))
    return ari.value, nmi.value


def spectral_cluster(n, src, dst, method, X0, n_clusters, init_rows, *, max_iters,
                     dtype="f64", km_max_iters=100, reorder=None, comm: Comm | None = None,
                     stream=None, **run_opts):
    """Algorithm 1 end to end from host buffers (ofsc_spectral_cluster).

    X0: host (n x k) array, original node order (copied; features returned).
    Returns (labels int32[n], features, report); with several ranks each rank
    fills the entries of the nodes it owns."""
    npdt = np.float64 if dtype == "f64" else np.float32
    X = np.ascontiguousarray(np.array(X0, dtype=npdt))
    src = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
    dst = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
    rows = np.ascontiguousarray(np.asarray(init_rows, dtype=np.int64))
    labels = np.full(X.shape[0], -1, np.int32)
    o = make_opts(X.shape[1], max_iters, **run_opts)
    bo = None if reorder is None else BuildOpts(1 if reorder else 0, 30)   # None: library default
    rep = Report()
    _check(lib().ofsc_spectral_cluster(comm.handle if comm else None, int(n), src.size,
                                       src.ctypes.data_as(C.c_void_p),
                                       dst.ctypes.data_as(C.c_void_p), METHODS[method],
                                       DTYPES[dtype], C.byref(o), C.byref(bo) if bo else None,
                                       X.ctypes.data_as(C.c_void_p), int(n_clusters),
                                       rows.ctypes.data_as(C.c_void_p), int(km_max_iters),
                                       labels.ctypes.data_as(C.c_void_p), C.byref(rep),
                                       _stream(stream) if stream is not None else None))
    return labels, X, rep.as_dict()

// libofsc C ABI and host runtime: graph handles, workspaces, the iteration
// schedule (captured once as a CUDA graph per iteration kind), NCCL
// collectives for the row-partitioned multi-GPU path, K-means driver, scores.
// See include/ofsc.h for the contract of every entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include "internal.h"

namespace ofsc {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

template <typename F>
static ofsc_status guard(F&& f) {
  try {
    f();
    return OFSC_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.st;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return OFSC_ERR_NOMEM;
  } catch (...) {
    set_last_error("unknown internal error");
    return OFSC_ERR_STATE;
  }
}

static size_t esize(ofsc_dtype dt) { return dt == OFSC_F64 ? 8 : 4; }

// RAII device buffer (stream-ordered allocation)
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) dev_alloc(&p, bytes, st);
  }
  ~DBuf() { release(); }
  void release() {
    dev_free_async(p, s);
    p = nullptr;
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  template <typename T>
  T* as() const { return (T*)p; }
};

static void dfree(void* p) { dev_free(p); }

static ncclDataType_t nccl_type(ofsc_dtype dt) { return dt == OFSC_F64 ? ncclFloat64 : ncclFloat32; }

// Per-graph run workspace (allocated on first run, reused while (dtype, KP) match).
struct Workspace {
  bool have = false;
  ofsc_dtype dt = OFSC_F64;
  int KP = 0;
  void *X = nullptr, *AX = nullptr, *G = nullptr, *AV = nullptr, *Vg = nullptr, *Xg = nullptr;
  void* sendbuf = nullptr;  // p > 1: packed rows of the halo exchange
  cudaStream_t comm_st = nullptr;            // p > 1: halo exchange overlapped with the SpMM
  cudaEvent_t ev_v = nullptr, ev_x = nullptr;
  cudaStream_t fork_st = nullptr;            // p == 1: C4's Gram reduction beside the SpMM
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr;
  double *part_cols = nullptr, *part_g4 = nullptr, *part_g2 = nullptr, *grams = nullptr;
  double* part_gd = nullptr;  // f1 methods: column dots diag T, diag R' per block
  double* state = nullptr;  // M, W [KP*KP each], alpha, beta, gg_prev [KP], colred, diagred [2KP]
  DevCtl* ctl = nullptr;
  unsigned long long* ctr = nullptr;  // SpMM work counter
  int nb3 = 0, nb4 = 0, nb2 = 0, nbd = 0;
  cudaGraph_t g_iter = nullptr, g_refresh = nullptr, g_loop = nullptr;
  cudaGraphExec_t e_iter = nullptr, e_refresh = nullptr, e_loop = nullptr;
  cudaStream_t cap = nullptr;  // private stream used only for graph capture
  void release() {
    if (have) cudaDeviceSynchronize();   // pool frees below: no queued user left
    if (cap) cudaStreamDestroy(cap);
    cap = nullptr;
    if (comm_st) cudaStreamDestroy(comm_st);
    if (ev_v) cudaEventDestroy(ev_v);
    if (ev_x) cudaEventDestroy(ev_x);
    comm_st = nullptr;
    ev_v = ev_x = nullptr;
    if (fork_st) cudaStreamDestroy(fork_st);
    if (ev_f0) cudaEventDestroy(ev_f0);
    if (ev_f1) cudaEventDestroy(ev_f1);
    fork_st = nullptr;
    ev_f0 = ev_f1 = nullptr;
    if (e_iter) cudaGraphExecDestroy(e_iter);
    if (e_refresh) cudaGraphExecDestroy(e_refresh);
    if (e_loop) cudaGraphExecDestroy(e_loop);
    if (g_iter) cudaGraphDestroy(g_iter);
    if (g_refresh) cudaGraphDestroy(g_refresh);
    if (g_loop) cudaGraphDestroy(g_loop);
    e_iter = e_refresh = e_loop = nullptr;
    g_iter = g_refresh = g_loop = nullptr;
    for (void* q : {X, AX, G, AV, Vg, Xg, sendbuf, (void*)part_cols, (void*)part_g4, (void*)part_g2,
                    (void*)part_gd, (void*)grams, (void*)state, (void*)ctl, (void*)ctr})
      dfree(q);
    ctr = nullptr;
    X = AX = G = AV = Vg = Xg = sendbuf = nullptr;
    part_cols = part_g4 = part_g2 = part_gd = grams = state = nullptr;
    ctl = nullptr;
    have = false;
  }
};

}  // namespace ofsc

using namespace ofsc;

struct ofsc_graph_s {
  ofsc_comm comm = nullptr;
  int p = 1, rank = 0;
  int64_t n = 0, row_begin = 0, row_end = 0, n_local = 0, slot_rows = 0, own_off = 0;
  int64_t nnz_local = 0;
  std::vector<int64_t> begins;     // p + 1
  int64_t* d_begins = nullptr;
  int64_t* row_ptr = nullptr;      // n_local + 1, from 0
  int32_t* col = nullptr;          // gather-buffer row ids (== global ids when p == 1)
  double* s_slot = nullptr;        // s on the gather rows: [n] (p == 1) or [ext_rows] (halo)
  float* s32_slot = nullptr;
  int32_t* perm = nullptr;         // internal row -> original node (reordered graphs)
  // gather layout (p > 1: halo layout, graph_build.cu build_halo): ext rows = own rows then
  // the remote rows this rank's columns reference; the SpMM gathers from a buffer of ext_rows
  int64_t ext_rows = 0;
  int32_t* d_gid = nullptr;        // [ext_rows] global id of each ext row (NULL when p == 1)
  std::vector<int32_t> h_gid;
  std::vector<int64_t> recv_cnt, recv_off, send_cnt, send_off;
  int32_t* d_send_idx = nullptr;   // own rows to send, grouped by peer
  int64_t total_send = 0;
  double* red_gather = nullptr;    // p > 1: [p][4 KP^2] scratch of the rank-order sums (comm.cu)
  // the local CSR split per row: own-row columns | halo columns (p > 1, for the overlap)
  int64_t* row_ptr_loc = nullptr;
  int32_t* col_loc = nullptr;
  int64_t* row_ptr_rem = nullptr;
  int32_t* col_rem = nullptr;
  int32_t* cid = nullptr;          // community of each internal row (reordered graphs)
  int64_t* cstart = nullptr;       // community start rows [n_comm + 1]
  HeavyRows heavy, heavy_loc, heavy_rem;  // power-law rows split into chunks (SpMM binning)
  SvalStream svs;                  // neighbour-scale stream of the SpMM (p == 1, large graphs)
  bool reordered = false;
  ofsc_graph_info info{};
  Workspace ws;
  // permutation applied at the user boundary (p == 1 only; p > 1 uses internal order)
  const int32_t* user_perm() const { return (reordered && p == 1) ? perm : nullptr; }
};

extern "C" {

const char* ofsc_version(void) { return "ofsc 0.1.0 (sm_100a)"; }

ofsc_status ofsc_trim_memory(void) {
  return guard([&] { dev_trim(); });
}

const char* ofsc_status_string(ofsc_status s) {
  switch (s) {
    case OFSC_OK: return "ok";
    case OFSC_ERR_ARG: return "invalid argument";
    case OFSC_ERR_RANGE: return "edge endpoint out of range";
    case OFSC_ERR_NOMEM: return "out of memory";
    case OFSC_ERR_CUDA: return "CUDA error";
    case OFSC_ERR_NCCL: return "NCCL error";
    case OFSC_ERR_DIVERGED: return "iteration diverged (non-finite direction or step)";
    case OFSC_ERR_STATE: return "invalid state";
  }
  return "unknown status";
}

const char* ofsc_last_error(void) { return g_last_error.c_str(); }

void ofsc_opts_default(ofsc_opts* o) {
  if (!o) return;
  o->k = 0;
  o->max_iters = 100;
  o->tol = 0.0;
  o->beta_rule = OFSC_BETA_PR_PLUS;
  o->line_search = 1;
  o->alpha_fixed = 0.0;
  o->refresh = 0;
  o->check_every = 8;
  o->timing_skip = -1;
  o->profile = 0;
}

ofsc_status ofsc_get_unique_id(void* h_id128) {
  return guard([&] {
    OFSC_REQUIRE(h_id128, OFSC_ERR_ARG, "null id");
    static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
    ncclUniqueId id;
    OFSC_NCCL(ncclGetUniqueId(&id));
    std::memcpy(h_id128, &id, 128);
  });
}

ofsc_status ofsc_comm_create(const void* h_id128, int nranks, int rank, int cuda_device,
                             ofsc_comm* out) {
  return guard([&] {
    OFSC_REQUIRE(h_id128 && out && nranks >= 1 && rank >= 0 && rank < nranks, OFSC_ERR_ARG,
                 "bad communicator arguments");
    OFSC_CUDA(cudaSetDevice(cuda_device));
    auto* c = new ofsc_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->device = cuda_device;
    ncclUniqueId id;
    std::memcpy(&id, h_id128, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      throw Error{OFSC_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)};
    }
    *out = c;
  });
}

ofsc_status ofsc_comm_destroy(ofsc_comm comm) {
  return guard([&] {
    if (!comm) return;
    if (comm->nccl) ncclCommDestroy(comm->nccl);
    delete comm;
  });
}

// ---------------------------------------------------------------------------
// graph build
// ---------------------------------------------------------------------------
// Contiguous split of rows [0, n) over p ranks with ~equal nnz(A) = sum (deg_i + 1).
static void partition_rows(int64_t n, const int64_t* rp, int p, int64_t* begins) {
  begins[0] = 0;
  begins[p] = n;
  const double total = (double)(rp[n] + n);
  int64_t i = 0;
  for (int r = 1; r < p; ++r) {
    const double target = total * r / p;
    while (i < n && (double)(rp[i] + i) < target) ++i;
    begins[r] = std::max(i, begins[r - 1]);
  }
}

ofsc_status ofsc_partition_rows(int64_t n, const int64_t* h_row_ptr, int p, int64_t* h_begins) {
  return guard([&] {
    OFSC_REQUIRE(n >= 1 && h_row_ptr && h_begins && p >= 1, OFSC_ERR_ARG, "bad partition args");
    partition_rows(n, h_row_ptr, p, h_begins);
  });
}

ofsc_status ofsc_comm_create_local_world(int nranks, ofsc_comm* out) {
  return guard([&] {
    OFSC_REQUIRE(out && nranks >= 1, OFSC_ERR_ARG, "bad communicator arguments");
    int dev = 0;
    OFSC_CUDA(cudaGetDevice(&dev));
    auto world = make_local_world(nranks);
    for (int r = 0; r < nranks; ++r) {
      auto* c = new ofsc_comm_s();
      c->nranks = nranks;
      c->rank = r;
      c->device = dev;
      c->world = world;
      out[r] = c;
    }
  });
}

ofsc_status ofsc_comm_create_local(int nranks, int rank, ofsc_comm* out) {
  return guard([&] {
    OFSC_REQUIRE(out && nranks >= 1 && rank >= 0 && rank < nranks, OFSC_ERR_ARG,
                 "bad communicator arguments");
    auto* c = new ofsc_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    OFSC_CUDA(cudaGetDevice(&c->device));
    *out = c;  // nccl == nullptr: no collectives (test communicator)
  });
}

static void graph_free(ofsc_graph g) {
  cudaDeviceSynchronize();   // nothing queued may still use the buffers (pool frees follow)
  g->ws.release();
  dfree(g->d_begins);
  dfree(g->row_ptr);
  dfree(g->col);
  dfree(g->s_slot);
  dfree(g->s32_slot);
  dfree(g->perm);
  dfree(g->cid);
  dfree(g->cstart);
  dfree(g->d_gid);
  dfree(g->d_send_idx);
  dfree(g->red_gather);
  dfree(g->row_ptr_loc);
  dfree(g->col_loc);
  dfree(g->row_ptr_rem);
  dfree(g->col_rem);
  g->heavy.release();
  g->heavy_loc.release();
  g->heavy_rem.release();
  g->svs.release();
}

ofsc_status ofsc_graph_build(ofsc_comm comm, int64_t n, int64_t m, const int64_t* src,
                             const int64_t* dst, int edges_on_device, ofsc_stream stream,
                             ofsc_graph* out) {
  return ofsc_graph_build_ex(comm, n, m, src, dst, edges_on_device, nullptr, stream, out);
}

ofsc_status ofsc_graph_build_ex(ofsc_comm comm, int64_t n, int64_t m, const int64_t* src,
                                const int64_t* dst, int edges_on_device,
                                const ofsc_build_opts* bopts, ofsc_stream stream,
                                ofsc_graph* out) {
  ofsc_graph g = nullptr;
  ofsc_status st = guard([&] {
    OFSC_REQUIRE(out && n >= 1 && m >= 0 && (m == 0 || (src && dst)), OFSC_ERR_ARG,
                 "bad graph arguments");
    const int reorder = bopts ? bopts->reorder : 0;
    const int sweeps = (bopts && bopts->lpa_sweeps > 0) ? bopts->lpa_sweeps : 30;
    OFSC_REQUIRE(reorder == 0 || reorder == 1, OFSC_ERR_ARG, "bad reorder option");
    cudaStream_t s = (cudaStream_t)stream;
    g = new ofsc_graph_s();
    g->comm = comm;
    g->p = comm ? comm->nranks : 1;
    g->rank = comm ? comm->rank : 0;
    g->n = n;
    CsrDevice csr;
    int64_t n_comm = 0;
    double intra = 0.0;
    auto free_csr = [&] {   // stream-ordered pool frees: no device-wide synchronisation
      dev_free_async(csr.row_ptr, s);
      dev_free_async(csr.col, s);
      dev_free_async(csr.s, s);
      csr.row_ptr = nullptr;
      csr.col = nullptr;
      csr.s = nullptr;
    };
    {
      const size_t eb = (!edges_on_device && m > 0) ? m * sizeof(int64_t) : 0;
      DBuf ds(eb, s), dd(eb, s);
      const int64_t* psrc = src;
      const int64_t* pdst = dst;
      if (eb) {
        OFSC_CUDA(cudaMemcpyAsync(ds.p, src, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        OFSC_CUDA(cudaMemcpyAsync(dd.p, dst, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        psrc = ds.as<int64_t>();
        pdst = dd.as<int64_t>();
      }
      trace_point("graph_build: edges on device", s);
      try {
        build_csr(n, m, psrc, pdst, csr, s);
        if (reorder) {
          // locality reordering derived from the graph: communities -> contiguous rows
          dev_alloc((void**)&g->perm, n * sizeof(int32_t), s);
          dev_alloc((void**)&g->cid, n * sizeof(int32_t), s);
          DBuf inv(n * sizeof(int32_t), s);
          lpa_order(csr, sweeps, g->perm, inv.as<int32_t>(), &n_comm, &intra, g->cid, &g->cstart, s);
          DBuf s2(m * sizeof(int64_t), s), d2(m * sizeof(int64_t), s);
          trace_point("graph_build: LPA order", s);
          relabel_edges(m, n, psrc, pdst, inv.as<int32_t>(), s2.as<int64_t>(), d2.as<int64_t>(), s);
          free_csr();
          build_csr(n, m, s2.as<int64_t>(), d2.as<int64_t>(), csr, s);
          g->reordered = true;
        }
      } catch (...) {
        free_csr();
        throw;
      }
    }
    const int p = g->p;
    // nnz-balanced contiguous row split (each row weighted deg + 1: nnz(A) incl. diagonal)
    // p == 1 needs only row_ptr[0] = 0 and row_ptr[n] = nnz (no 8(n+1)-byte download)
    std::vector<int64_t> rp(p == 1 ? 0 : n + 1);
    if (p > 1) {
      OFSC_CUDA(cudaMemcpyAsync(rp.data(), csr.row_ptr, (n + 1) * sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
    }
    OFSC_CUDA(cudaStreamSynchronize(s));
    trace_point("graph_build: row_ptr on host", s);
    auto rp_at = [&](int64_t i) -> int64_t { return p == 1 ? (i == 0 ? 0 : csr.nnz) : rp[i]; };
    g->begins.assign(p + 1, 0);
    if (p == 1) g->begins[1] = n;
    else partition_rows(n, rp.data(), p, g->begins.data());
    const double total = (double)(csr.nnz + n);
    g->row_begin = g->begins[g->rank];
    g->row_end = g->begins[g->rank + 1];
    g->n_local = g->row_end - g->row_begin;
    int64_t max_nnz = 0;
    for (int r = 0; r < p; ++r) {
      const int64_t nz = rp_at(g->begins[r + 1]) - rp_at(g->begins[r]) + (g->begins[r + 1] - g->begins[r]);
      max_nnz = std::max(max_nnz, nz);
    }
    g->slot_rows = n;     // p == 1: the gather buffer is the whole X (p > 1: set below)
    g->own_off = 0;
    g->ext_rows = n;
    const int64_t e0 = rp_at(g->row_begin), e1 = rp_at(g->row_end);
    g->nnz_local = e1 - e0;
    if (p == 1) {
      g->row_ptr = csr.row_ptr;
      g->col = csr.col;
      g->s_slot = csr.s;
      dev_alloc((void**)&g->s32_slot, n * sizeof(float), s);
      dev_alloc((void**)&g->d_begins, 2 * sizeof(int64_t), s);
      OFSC_CUDA(cudaMemcpyAsync(g->d_begins, g->begins.data(), 2 * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
      scatter_slots(csr.s, n, g->s_slot, g->s32_slot, g->d_begins, 1, n, s);
    } else {
      dev_alloc((void**)&g->d_begins, (p + 1) * sizeof(int64_t), s);
      OFSC_CUDA(cudaMemcpyAsync(g->d_begins, g->begins.data(), (p + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
      HaloLayout hl;
      try {
        build_halo(csr, g->begins.data(), g->d_begins, p, g->rank, hl, s);
      } catch (...) {
        dfree(hl.row_ptr); dfree(hl.col); dfree(hl.s_ext); dfree(hl.s32_ext);
        dfree(hl.d_gid); dfree(hl.d_send_idx);
        dfree(hl.row_ptr_loc); dfree(hl.col_loc); dfree(hl.row_ptr_rem); dfree(hl.col_rem);
        free_csr();
        throw;
      }
      g->row_ptr = hl.row_ptr;
      g->col = hl.col;
      g->s_slot = hl.s_ext;
      g->s32_slot = hl.s32_ext;
      g->d_gid = hl.d_gid;
      g->h_gid = std::move(hl.h_gid);
      g->ext_rows = hl.ext_rows;
      g->recv_cnt = hl.recv_cnt;
      g->recv_off = hl.recv_off;
      g->send_cnt = hl.send_cnt;
      g->send_off = hl.send_off;
      g->d_send_idx = hl.d_send_idx;
      g->total_send = hl.total_send;
      g->row_ptr_loc = hl.row_ptr_loc;
      g->col_loc = hl.col_loc;
      g->row_ptr_rem = hl.row_ptr_rem;
      g->col_rem = hl.col_rem;
      g->own_off = 0;
      g->slot_rows = hl.ext_rows;
      dev_alloc((void**)&g->red_gather, (size_t)p * 4 * OFSC_MAX_K * OFSC_MAX_K * sizeof(double), s);
      OFSC_CUDA(cudaStreamSynchronize(s));
      build_heavy(g->row_ptr_loc, g->n_local, g->heavy_loc, s);
      build_heavy(g->row_ptr_rem, g->n_local, g->heavy_rem, s);
      free_csr();
    }
    OFSC_CUDA(cudaStreamSynchronize(s));
    ofsc_graph_info& in = g->info;
    in.n = n;
    in.n_edges_kept = csr.m_kept;
    in.nnz_global = csr.nnz;
    in.row_begin = g->row_begin;
    in.row_end = g->row_end;
    in.nnz_local = g->nnz_local;
    in.n_isolated = csr.n_isolated;
    in.n_self_loops_dropped = csr.n_loops;
    in.n_duplicates_dropped = csr.n_dups;
    in.max_degree = csr.max_deg;
    in.fro2_A = csr.fro2;
    in.load_imbalance = (double)p * (double)max_nnz / total;
    in.reordered = g->reordered ? 1 : 0;
    in.n_communities = n_comm;
    in.intra_edge_fraction = intra;
    build_heavy(g->row_ptr, g->n_local, g->heavy, s);
    if (p == 1)
      build_sval(n, g->nnz_local, g->row_ptr, g->col, g->s_slot, g->s32_slot, in.max_degree,
                 g->svs, s);
    in.halo_rows = g->ext_rows - g->n_local;
    in.send_rows = g->total_send;
    trace_point("graph_build: done", s);
    *out = g;
  });
  if (st != OFSC_OK && g) {
    graph_free(g);
    delete g;
  }
  return st;
}

__global__ void k_invert_perm_b(int64_t n, const int32_t* perm, int32_t* inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

ofsc_status ofsc_graph_append(ofsc_graph g, int64_t m, const int64_t* src, const int64_t* dst,
                              int edges_on_device, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(g && m >= 0 && (m == 0 || (src && dst)), OFSC_ERR_ARG, "bad append arguments");
    OFSC_REQUIRE(g->p == 1, OFSC_ERR_STATE,
                 "ofsc_graph_append supports single-rank graphs (rebuild for p > 1)");
    if (m == 0) return;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = g->n;
    const size_t eb = (size_t)m * sizeof(int64_t);
    DBuf ds(edges_on_device ? 0 : eb, s), dd(edges_on_device ? 0 : eb, s);
    const int64_t* psrc = src;
    const int64_t* pdst = dst;
    if (!edges_on_device) {
      OFSC_CUDA(cudaMemcpyAsync(ds.p, src, eb, cudaMemcpyHostToDevice, s));
      OFSC_CUDA(cudaMemcpyAsync(dd.p, dst, eb, cudaMemcpyHostToDevice, s));
      psrc = ds.as<int64_t>();
      pdst = dd.as<int64_t>();
    }
    DBuf s2(g->reordered ? eb : 0, s), d2(g->reordered ? eb : 0, s), inv(g->reordered ? n * 4 : 0, s);
    if (g->reordered) {   // original ids -> internal (community-ordered) rows; the order is kept
      k_invert_perm_b<<<num_sms() * 8, 256, 0, s>>>(n, g->perm, inv.as<int32_t>());
      OFSC_LAUNCH_CHECK();
      relabel_edges(m, n, psrc, pdst, inv.as<int32_t>(), s2.as<int64_t>(), d2.as<int64_t>(), s);
      psrc = s2.as<int64_t>();
      pdst = d2.as<int64_t>();
    }
    CsrDevice csr;
    csr.n = n;
    csr.row_ptr = g->row_ptr;
    csr.col = g->col;
    csr.s = g->s_slot;
    csr.nnz = g->info.nnz_global;
    csr.m_kept = g->info.n_edges_kept;
    csr.n_loops = g->info.n_self_loops_dropped;
    csr.n_dups = g->info.n_duplicates_dropped;
    csr.n_isolated = g->info.n_isolated;
    csr.max_deg = g->info.max_degree;
    csr.fro2 = g->info.fro2_A;
    g->ws.release();                 // captured iteration graphs hold the old CSR pointers
    append_csr(csr, m, psrc, pdst, s);
    g->row_ptr = csr.row_ptr;
    g->col = csr.col;
    scatter_slots(csr.s, n, g->s_slot, g->s32_slot, g->d_begins, 1, n, s);
    build_heavy(g->row_ptr, n, g->heavy, s);
    build_sval(n, csr.nnz, g->row_ptr, g->col, g->s_slot, g->s32_slot, csr.max_deg, g->svs, s);
    OFSC_CUDA(cudaStreamSynchronize(s));
    g->nnz_local = csr.nnz;
    ofsc_graph_info& in = g->info;
    in.n_edges_kept = csr.m_kept;
    in.nnz_global = csr.nnz;
    in.nnz_local = csr.nnz;
    in.n_isolated = csr.n_isolated;
    in.n_self_loops_dropped = csr.n_loops;
    in.n_duplicates_dropped = csr.n_dups;
    in.max_degree = csr.max_deg;
    in.fro2_A = csr.fro2;
  });
}

ofsc_status ofsc_graph_exchange_plan(ofsc_graph g, int64_t* h_send_counts, int32_t* h_send_gids,
                                     int64_t* h_recv_counts, int32_t* h_recv_gids) {
  return guard([&] {
    OFSC_REQUIRE(g, OFSC_ERR_ARG, "null graph");
    for (int q = 0; q < g->p; ++q) {
      if (h_send_counts) h_send_counts[q] = g->p > 1 ? g->send_cnt[q] : 0;
      if (h_recv_counts) h_recv_counts[q] = g->p > 1 ? g->recv_cnt[q] : 0;
    }
    if (g->p == 1) return;
    if (h_send_gids && g->total_send > 0) {
      std::vector<int32_t> idx(g->total_send);
      OFSC_CUDA(cudaMemcpy(idx.data(), g->d_send_idx, idx.size() * sizeof(int32_t),
                           cudaMemcpyDeviceToHost));
      for (int64_t t = 0; t < g->total_send; ++t) h_send_gids[t] = (int32_t)(g->row_begin + idx[t]);
    }
    if (h_recv_gids)
      for (int64_t e = g->n_local; e < g->ext_rows; ++e) h_recv_gids[e - g->n_local] = g->h_gid[e];
  });
}

ofsc_status ofsc_graph_info_get(ofsc_graph g, ofsc_graph_info* out) {
  return guard([&] {
    OFSC_REQUIRE(g && out, OFSC_ERR_ARG, "null argument");
    *out = g->info;
  });
}

ofsc_status ofsc_graph_copy_csr(ofsc_graph g, int64_t* h_row_ptr, int32_t* h_col, double* h_s) {
  return guard([&] {
    OFSC_REQUIRE(g, OFSC_ERR_ARG, "null graph");
    if (h_row_ptr)
      OFSC_CUDA(cudaMemcpy(h_row_ptr, g->row_ptr, (g->n_local + 1) * sizeof(int64_t),
                           cudaMemcpyDeviceToHost));
    if (h_col && g->nnz_local > 0) {
      OFSC_CUDA(cudaMemcpy(h_col, g->col, g->nnz_local * sizeof(int32_t), cudaMemcpyDeviceToHost));
      if (g->p > 1)    // ext ids -> global ids
        for (int64_t e = 0; e < g->nnz_local; ++e) h_col[e] = g->h_gid[h_col[e]];
    }
    if (h_s) {
      if (g->p == 1) {
        OFSC_CUDA(cudaMemcpy(h_s, g->s_slot, g->n * sizeof(double), cudaMemcpyDeviceToHost));
      } else {   // s of the rows this rank sees (own + halo); other entries are not held here
        std::vector<double> ext(g->ext_rows);
        OFSC_CUDA(cudaMemcpy(ext.data(), g->s_slot, ext.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        for (int64_t q = 0; q < g->n; ++q) h_s[q] = 0.0;
        for (int64_t e = 0; e < g->ext_rows; ++e) h_s[g->h_gid[e]] = ext[e];
      }
    }
  });
}

ofsc_status ofsc_graph_copy_perm(ofsc_graph g, int32_t* h_perm) {
  return guard([&] {
    OFSC_REQUIRE(g && h_perm, OFSC_ERR_ARG, "null argument");
    if (g->reordered)
      OFSC_CUDA(cudaMemcpy(h_perm, g->perm, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    else
      for (int64_t i = 0; i < g->n; ++i) h_perm[i] = (int32_t)i;
  });
}

ofsc_status ofsc_graph_destroy(ofsc_graph g) {
  return guard([&] {
    if (!g) return;
    cudaDeviceSynchronize();
    graph_free(g);
    delete g;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// helpers for the hooks: user layout (global rows, ld) -> gather-buffer layout (KP)
// ---------------------------------------------------------------------------
namespace ofsc {

// ext row e (global row gid[e], identity when gid == NULL) <- user row perm[gid]
__global__ void k_to_ext(int k, int KP, int64_t rows, const void* src, int64_t lds, void* dst,
                         const int32_t* gid, int f64, const int32_t* perm) {
  const int64_t total = rows * KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / KP;
    const int c = (int)(e % KP);
    const int64_t g = gid ? (int64_t)gid[r] : r;
    const int64_t u = perm ? (int64_t)perm[g] : g;
    if (f64) ((double*)dst)[r * KP + c] = c < k ? ((const double*)src)[u * lds + c] : 0.0;
    else ((float*)dst)[r * KP + c] = c < k ? ((const float*)src)[u * lds + c] : 0.0f;
  }
}

// full user array (all n rows, original order) -> this rank's gather buffer
static void to_slots(ofsc_graph g, ofsc_dtype dt, int k, int KP, const void* src, int64_t lds,
                     void* dst, cudaStream_t s) {
  k_to_ext<<<num_sms() * 8, 256, 0, s>>>(k, KP, g->ext_rows, src, lds, dst, g->d_gid,
                                         dt == OFSC_F64, g->reordered ? g->perm : nullptr);
  OFSC_LAUNCH_CHECK();
}

// Halo exchange (p > 1): pack the own rows each peer needs, then one grouped
// send/recv per peer into the peer's halo segment of the gather buffer.
__global__ void k_pack_rows(int64_t rows, int KP, const int32_t* idx, const void* src, void* dst,
                            int f64) {
  const int64_t total = rows * KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / KP, c = e % KP;
    const int64_t from = (int64_t)idx[r] * KP + c;
    if (f64) ((double*)dst)[e] = ((const double*)src)[from];
    else ((float*)dst)[e] = ((const float*)src)[from];
  }
}

static void halo_exchange(ofsc_graph g, ofsc_dtype dt, int KP, void* ext, void* sendbuf,
                          cudaStream_t s) {
  if (!comm_active(g->comm)) return;   // a bare local test communicator has no transport
  if (g->total_send > 0) {
    k_pack_rows<<<num_sms() * 8, 256, 0, s>>>(g->total_send, KP, g->d_send_idx, ext, sendbuf,
                                             dt == OFSC_F64);
    OFSC_LAUNCH_CHECK();
  }
  comm_exchange(g->comm, nccl_type(dt), KP, esize(dt), sendbuf, g->send_cnt, g->send_off, ext,
                g->recv_cnt, g->recv_off, s);
}

// Sum over ranks of k x k partials (Grams, column dots): all-gather + rank-order sum
// (comm.cu), identical bits on every rank.  A bare local test communicator keeps
// rank-partial sums.
static void allreduce_d(ofsc_graph g, double* buf, size_t count, cudaStream_t s) {
  if (g->p > 1 && comm_active(g->comm)) {
    OFSC_REQUIRE(count <= (size_t)4 * OFSC_MAX_K * OFSC_MAX_K, OFSC_ERR_STATE, "reduction too large");
    comm_sum_f64(g->comm, buf, count, g->red_gather, s);
  }
}

__global__ void k_extract_kk(const double* in, int KP, int k, double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * k) out[e] = in[(e / k) * KP + (e % k)];
}
__global__ void k_embed_kk(const double* in, int KP, int k, double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < KP * KP) {
    const int i = e / KP, j = e % KP;
    out[e] = (i < k && j < k) ? in[i * k + j] : 0.0;
  }
}

}  // namespace ofsc

extern "C" {

ofsc_status ofsc_graph_apply(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_Z, int64_t ldz,
                             void* d_Y, int64_t ldy, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(g && d_Z && d_Y && k >= 1 && ldz >= k && ldy >= k, OFSC_ERR_ARG, "bad apply args");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    cudaStream_t s = (cudaStream_t)stream;
    if (k > OFSC_MAX_K) {   // wider than the iteration's kernels: one thread per (row, column)
      DBuf zs(g->p == 1 && !g->reordered ? 0 : (size_t)g->ext_rows * k * esize(dt), s);
      DBuf ys(g->user_perm() ? (size_t)std::max<int64_t>(g->n_local, 1) * k * esize(dt) : 0, s);
      const void* Z = d_Z;
      int64_t lz = ldz;
      if (zs.p) {
        to_slots(g, dt, k, k, d_Z, ldz, zs.p, s);
        Z = zs.p;
        lz = k;
      }
      launch_spmm_plain(dt, k, g->n_local, g->own_off, g->row_ptr, g->col, g->s_slot, g->s32_slot,
                        Z, lz, g->user_perm() ? ys.p : d_Y, g->user_perm() ? k : ldy, s);
      if (g->user_perm()) launch_copy_out(dt, k, k, g->n_local, ys.p, d_Y, ldy, g->user_perm(), s);
      return;
    }
    // the iteration's SpMM kernel (C2a: k_spmm, degree binning, s_j stream, and for
    // p > 1 the split own-column / halo-column passes) on KP-padded copies
    const int KP = padded_k(k);
    const size_t es = esize(dt);
    const int64_t nl = g->n_local;
    DBuf zs((size_t)g->ext_rows * KP * es, s), ys(std::max<int64_t>(nl, 1) * KP * es, s),
        ctr(4 * sizeof(unsigned long long), s);
    to_slots(g, dt, k, KP, d_Z, ldz, zs.p, s);
    if (g->p > 1) {
      launch_spmm(dt, KP, nl, 0, g->row_ptr_loc, g->col_loc, g->s_slot, g->s32_slot, zs.p, ys.p,
                  nullptr, s, nullptr, nullptr, ctr.as<unsigned long long>(), 1, &g->heavy_loc);
      launch_spmm(dt, KP, nl, 0, g->row_ptr_rem, g->col_rem, g->s_slot, g->s32_slot, zs.p, ys.p,
                  nullptr, s, nullptr, nullptr, ctr.as<unsigned long long>(), 2, &g->heavy_rem);
    } else {
      launch_spmm(dt, KP, nl, g->own_off, g->row_ptr, g->col, g->s_slot, g->s32_slot, zs.p, ys.p,
                  nullptr, s, nullptr, nullptr, ctr.as<unsigned long long>(), 0, &g->heavy,
                  &g->svs, g->nnz_local);
    }
    launch_copy_out(dt, k, KP, nl, ys.p, d_Y, ldy, g->user_perm(), s);
  });
}

ofsc_status ofsc_graph_apply_gram(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_Z,
                                  int64_t ldz, const void* d_X, int64_t ldx, void* d_Y,
                                  int64_t ldy, double* d_grams, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(g && d_Z && d_X && d_Y && d_grams && k >= 1 && k <= OFSC_MAX_K && ldz >= k &&
                     ldx >= k && ldy >= k,
                 OFSC_ERR_ARG, "bad apply_gram args");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    cudaStream_t s = (cudaStream_t)stream;
    const int KP = padded_k(k);
    const size_t es = esize(dt);
    const int64_t nl = g->n_local;
    DBuf zs((size_t)g->ext_rows * KP * es, s), xs(std::max<int64_t>(nl, 1) * KP * es, s),
        ys(std::max<int64_t>(nl, 1) * KP * es, s);
    to_slots(g, dt, k, KP, d_Z, ldz, zs.p, s);
    launch_copy_in(dt, k, KP, nl, d_X, ldx, xs.p, g->user_perm(), s);
    const int nb = grid_rows(std::max<int64_t>(nl, 1), 2);
    const int nb2 = gram_stream_grid(dt, KP, std::max<int64_t>(nl, 1));
    DBuf p4((size_t)nb * 2 * KP * KP * 8, s), p2((size_t)nb2 * 2 * KP * KP * 8, s),
        gr((size_t)4 * KP * KP * 8, s);
    const char* zown = (const char*)zs.p + (size_t)g->own_off * KP * es;
    launch_gram_pair(dt, KP, nl, zown, zown, xs.p, p4.as<double>(), nb, s);
    if (g->p > 1) {   // the iteration's split form: own-row columns, then halo columns
      launch_spmm(dt, KP, nl, 0, g->row_ptr_loc, g->col_loc, g->s_slot, g->s32_slot, zs.p, ys.p,
                  nullptr, s, nullptr, nullptr, nullptr, 1, &g->heavy_loc);
      launch_spmm(dt, KP, nl, 0, g->row_ptr_rem, g->col_rem, g->s_slot, g->s32_slot, zs.p, ys.p,
                  nullptr, s, nullptr, nullptr, nullptr, 2, &g->heavy_rem);
      launch_gram_stream(dt, KP, nl, zown, xs.p, ys.p, p2.as<double>(), 0, nullptr, nb2, s);
    } else {
      launch_spmm_then_gram(dt, KP, nl, g->own_off, g->row_ptr, g->col, g->s_slot, g->s32_slot, zs.p,
                       xs.p, ys.p, p2.as<double>(), 0, nullptr, nb2, s, &g->heavy);
    }
    launch_reduce_partials(p4.as<double>(), nb, 2 * KP * KP, gr.as<double>(), s);
    launch_reduce_partials(p2.as<double>(), nb2, 2 * KP * KP, gr.as<double>() + 2 * KP * KP, s);
    allreduce_d(g, gr.as<double>(), 4 * KP * KP, s);
    launch_copy_out(dt, k, KP, nl, ys.p, d_Y, ldy, g->user_perm(), s);
    for (int q = 0; q < 4; ++q)
      k_extract_kk<<<(k * k + 255) / 256, 256, 0, s>>>(gr.as<double>() + q * KP * KP, KP, k,
                                                       d_grams + q * k * k);
    OFSC_LAUNCH_CHECK();
    OFSC_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// the iteration
// ---------------------------------------------------------------------------
namespace ofsc {

static void ensure_workspace(ofsc_graph g, ofsc_dtype dt, int KP, cudaStream_t s) {
  Workspace& w = g->ws;
  if (w.have && w.dt == dt && w.KP == KP) return;
  w.release();
  const size_t es = esize(dt);
  const int64_t nl = std::max<int64_t>(g->n_local, 1);
  const size_t blk = (size_t)nl * KP * es;
  dev_alloc((void**)&w.X, blk, s);
  dev_alloc((void**)&w.AX, blk, s);
  dev_alloc((void**)&w.G, blk, s);
  dev_alloc((void**)&w.AV, blk, s);
  const size_t vg = g->p == 1 ? blk : (size_t)g->ext_rows * KP * es;
  dev_alloc((void**)&w.Vg, vg, s);
  if (g->p > 1) {
    dev_alloc((void**)&w.sendbuf, (size_t)std::max<int64_t>(g->total_send, 1) * KP * es, s);
    OFSC_CUDA(cudaStreamCreateWithFlags(&w.comm_st, cudaStreamNonBlocking));
    OFSC_CUDA(cudaEventCreateWithFlags(&w.ev_v, cudaEventDisableTiming));
    OFSC_CUDA(cudaEventCreateWithFlags(&w.ev_x, cudaEventDisableTiming));
  }
  if (g->p == 1) {
    OFSC_CUDA(cudaStreamCreateWithFlags(&w.fork_st, cudaStreamNonBlocking));
    OFSC_CUDA(cudaEventCreateWithFlags(&w.ev_f0, cudaEventDisableTiming));
    OFSC_CUDA(cudaEventCreateWithFlags(&w.ev_f1, cudaEventDisableTiming));
  }
  const int nbmax = num_sms() * 4;   // grids of the streaming kernels are chosen per run
  w.nb2 = gram_stream_grid(dt, KP, nl);
  dev_alloc((void**)&w.part_cols, (size_t)nbmax * 2 * KP * 8, s);
  dev_alloc((void**)&w.part_g4, (size_t)nbmax * 2 * KP * KP * 8, s);
  dev_alloc((void**)&w.part_g2, (size_t)w.nb2 * 2 * KP * KP * 8, s);
  w.nbd = gram_diag_grid(nl);
  dev_alloc((void**)&w.part_gd, (size_t)w.nbd * 2 * KP * 8, s);
  dev_alloc((void**)&w.grams, (size_t)4 * KP * KP * 8, s);
  dev_alloc((void**)&w.state, (size_t)(2 * KP * KP + 7 * KP) * 8, s);
  dev_alloc((void**)&w.ctl, sizeof(DevCtl), s);
  dev_alloc((void**)&w.ctr, 4 * sizeof(unsigned long long), s);  // one per SpMM column pass
  w.dt = dt;
  w.KP = KP;
  w.have = true;
}

static IterParams make_params(ofsc_graph g, int method, const ofsc_opts& o, int KP) {
  Workspace& w = g->ws;
  w.nb3 = c3_grid(w.dt, KP, method, std::max<int64_t>(g->n_local, 1));
  w.nb4 = c4_grid(w.dt, KP, std::max<int64_t>(g->n_local, 1));
  const size_t es = esize(w.dt);
  IterParams p{};
  p.n_local = g->n_local;
  p.own_off = g->own_off;
  p.k = o.k;
  p.KP = KP;
  p.method = method;
  p.beta_rule = o.beta_rule;
  p.line_search = o.line_search;
  p.T = o.max_iters;
  p.alpha_fixed = o.alpha_fixed;
  p.tol = o.tol;
  static const double cm[4] = {4.0, 1.0, 2.0, 1.0};
  p.cm = cm[method];
  p.fro2 = g->info.fro2_A;
  p.X = w.X;
  p.AX = w.AX;
  p.G = w.G;
  p.AV = w.AV;
  p.Vg = w.Vg;
  p.V = g->p == 1 ? w.Vg : (void*)((char*)w.Vg + (size_t)g->own_off * KP * es);
  p.row_ptr = g->row_ptr;
  p.col = g->col;
  p.s = g->s_slot;
  p.s32 = g->s32_slot;
  p.M = w.state;
  p.W = w.state + KP * KP;
  p.alpha = w.state + 2 * KP * KP;
  p.beta = p.alpha + KP;
  p.gg_prev = p.beta + KP;
  p.colred = p.gg_prev + KP;
  p.diagred = p.colred + 2 * KP;
  p.grams = w.grams;
  p.part_cols = w.part_cols;
  p.part_g4 = w.part_g4;
  p.part_g2 = w.part_g2;
  p.part_gd = w.part_gd;
  p.ctl = w.ctl;
  p.spmm_ctr = w.ctr;
  return p;
}

// Per-phase launch accounting and optional CUDA-event timing (opts.profile).
struct Prof {
  bool timing = false;
  cudaStream_t s = nullptr;
  int launches[OFSC_NUM_PHASES] = {};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  template <typename F>
  void ph(int id, int nlaunch, F&& f) {
    launches[id] += nlaunch;
    if (!timing) {
      f();
      return;
    }
    cudaEvent_t a, b;
    OFSC_CUDA(cudaEventCreate(&a));
    OFSC_CUDA(cudaEventCreate(&b));
    OFSC_CUDA(cudaEventRecord(a, s));
    f();
    OFSC_CUDA(cudaEventRecord(b, s));
    ev.push_back({id, {a, b}});
  }
  int total() const {
    int t = 0;
    for (int i = 0; i < OFSC_NUM_PHASES; ++i) t += i == OFSC_PH_COMM ? 0 : launches[i];
    return t;
  }
  void resolve(double* ms) {
    for (auto& e : ev) {
      float x = 0.f;
      OFSC_CUDA(cudaEventElapsedTime(&x, e.second.first, e.second.second));
      ms[e.first] += x;
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    ev.clear();
  }
  ~Prof() {
    for (auto& e : ev) {
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
  }
};

// AX = A X, M = X^T X, W = X^T A X (init and refresh).  X must be current.
static void refresh_ops(ofsc_graph g, ofsc_dtype dt, const IterParams& p, cudaStream_t s,
                        Prof& pr) {
  Workspace& w = g->ws;
  const size_t es = esize(dt);
  const void* Zg = w.X;
  if (g->p > 1) {
    if (!w.Xg) dev_alloc((void**)&w.Xg, (size_t)g->ext_rows * p.KP * es, s);
    pr.ph(OFSC_PH_COMM, 0, [&] {
      OFSC_CUDA(cudaMemcpyAsync(w.Xg, w.X, (size_t)g->n_local * p.KP * es,
                                cudaMemcpyDeviceToDevice, s));
      halo_exchange(g, dt, p.KP, w.Xg, w.sendbuf, s);
    });
    Zg = w.Xg;
  }
  pr.ph(OFSC_PH_REFRESH, 3, [&] {
    // p == 1: the iteration SpMM's in-order row hand-out and neighbour-scale stream
    launch_spmm_then_gram(dt, p.KP, g->n_local, g->own_off, g->row_ptr, g->col, g->s_slot,
                     g->s32_slot, Zg, nullptr, w.AX, w.part_g2, 1, &p.ctl->stop, w.nb2, s,
                     &g->heavy, g->p == 1 ? w.ctr : nullptr, g->p == 1 ? &g->svs : nullptr,
                     g->nnz_local);
    launch_reduce_partials(w.part_g2, w.nb2, 2 * p.KP * p.KP, p.M, s);  // M, W contiguous
  });
  pr.ph(OFSC_PH_COMM, 0, [&] { allreduce_d(g, p.M, 2 * (size_t)p.KP * p.KP, s); });
}

static bool overlap_exchange() {   // OFSC_NO_OVERLAP=1: exchange, then one SpMM pass
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("OFSC_NO_OVERLAP");
    env = (e && e[0] == '1') ? 0 : 1;
  }
  return env == 1;
}

// One iteration of Algorithm 2 (l.8-12), the R-mode schedule of DESIGN.md:
// C3 -> beta -> C4 -> [all-gather V] -> C2 -> Gram reduce -> [all-reduce] -> line search.
static bool pdl_ls() {   // OFSC_PDL_LS=0: the line-search kernel waits for C2b in full
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("OFSC_PDL_LS");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1;
}

// OFM-f1 / TriOFM-f1: C2b forms only diag T and diag R' (their cubics, eq:f1-derivative
// P:298-305 and eq:alphai-f1 P:315-322, read T and R' through T_ii and R'_ii, and
// neither direction reads W = X^T A X, whose off-diagonal is then left as the last
// refresh formed it).  OFSC_F1_DIAG=0: the full Gram pair for every method (A/B).
static bool f1_diag(int method) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("OFSC_F1_DIAG");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1 && (method == OFSC_OFM_F1 || method == OFSC_TRIOFM_F1);
}

static void iteration_ops(ofsc_graph g, ofsc_dtype dt, const IterParams& p, bool refresh,
                          cudaStream_t s, Prof& pr) {
  Workspace& w = g->ws;
  if (refresh) {
    pr.ph(OFSC_PH_REFRESH, 1, [&] { launch_update_x(dt, p, s); });
    refresh_ops(g, dt, p, s, pr);
    pr.ph(OFSC_PH_UPDATE_DIRECTION, 1, [&] { launch_update_direction(dt, p, 0, w.nb3, s); });
  } else {
    pr.ph(OFSC_PH_UPDATE_DIRECTION, 1, [&] { launch_update_direction(dt, p, 1, w.nb3, s); });
  }
  // programmatic dependent launches along C3 -> beta -> C4 -> SpMM -> C2b (p == 1; not
  // in profiling runs, whose events sit between the launches): each kernel is
  // scheduled while its predecessor drains and waits in griddepcontrol.wait
  const bool pdl = g->p == 1 && !pr.timing;
  if (g->p == 1) {
    pdl_next(pdl);
    pr.ph(OFSC_PH_BETA, 1, [&] { launch_beta(p, w.nb3, 0, s); });
  } else {
    pr.ph(OFSC_PH_BETA, 1, [&] { launch_reduce_cols(p, w.nb3, s); });
    pr.ph(OFSC_PH_COMM, 0, [&] { allreduce_d(g, p.colred, 2 * (size_t)p.KP, s); });
    pr.ph(OFSC_PH_BETA, 1, [&] { launch_beta(p, w.nb3, 1, s); });
  }
  pdl_next(pdl);
  pr.ph(OFSC_PH_DIRECTION_GRAM, 1, [&] { launch_direction_gram(dt, p, w.nb4, s); });
  // p == 1: C4's partial Grams (Q, P) are reduced on a forked stream while the SpMM
  // and C2b run; the line search joins it (off the critical path)
  const bool fork_reduce = g->p == 1 && w.fork_st && !pr.timing;
  if (fork_reduce)
    pr.ph(OFSC_PH_GRAM_REDUCE, 1, [&] {
      OFSC_CUDA(cudaEventRecord(w.ev_f0, s));
      OFSC_CUDA(cudaStreamWaitEvent(w.fork_st, w.ev_f0, 0));
      launch_reduce_partials(w.part_g4, w.nb4, 2 * p.KP * p.KP, w.grams, w.fork_st);
      OFSC_CUDA(cudaEventRecord(w.ev_f1, w.fork_st));
    });
  if (g->p > 1 && overlap_exchange() && !pr.timing) {
    // halo exchange on the comm stream while the SpMM sums the own-row columns;
    // the halo columns are added once the exchange lands
    OFSC_CUDA(cudaEventRecord(w.ev_v, s));
    OFSC_CUDA(cudaStreamWaitEvent(w.comm_st, w.ev_v, 0));
    halo_exchange(g, dt, p.KP, w.Vg, w.sendbuf, w.comm_st);
    OFSC_CUDA(cudaEventRecord(w.ev_x, w.comm_st));
    pr.ph(OFSC_PH_SPMM_GRAM, 2, [&] {
      launch_spmm(dt, p.KP, g->n_local, 0, g->row_ptr_loc, g->col_loc, g->s_slot, g->s32_slot,
                  w.Vg, w.AV, &p.ctl->stop, s, nullptr, nullptr, w.ctr, 1, &g->heavy_loc);
      OFSC_CUDA(cudaStreamWaitEvent(s, w.ev_x, 0));
      launch_spmm(dt, p.KP, g->n_local, 0, g->row_ptr_rem, g->col_rem, g->s_slot, g->s32_slot,
                  w.Vg, w.AV, &p.ctl->stop, s, nullptr, nullptr, w.ctr, 2, &g->heavy_rem);
    });
  } else {
    if (g->p > 1)
      pr.ph(OFSC_PH_COMM, 0, [&] {
        halo_exchange(g, dt, p.KP, w.Vg, w.sendbuf, s);
      });
    pdl_next(pdl);
    pr.ph(OFSC_PH_SPMM_GRAM, 1, [&] {
      launch_spmm(dt, p.KP, g->n_local, g->own_off, g->row_ptr, g->col, g->s_slot, g->s32_slot,
                  w.Vg, w.AV, &p.ctl->stop, s, g->p == 1 ? g->cid : nullptr,
                  g->p == 1 ? g->cstart : nullptr, w.ctr, 0, &g->heavy,
                  g->p == 1 ? &g->svs : nullptr, g->nnz_local);
    });
  }
  pdl_next(pdl);
  // the f1 methods need only diag T, diag R' (k_gram_diag: 3B streamed, no k x k products)
  const bool diag = f1_diag(p.method);
  pr.ph(OFSC_PH_GRAM_STREAM, 1, [&] {
    if (diag)
      launch_gram_diag(dt, p.KP, g->n_local, p.V, w.X, w.AV, w.part_gd, &p.ctl->stop, w.nbd, s);
    else
      launch_gram_stream(dt, p.KP, g->n_local, p.V, w.X, w.AV, w.part_g2, 0, &p.ctl->stop, w.nb2, s);
  });
  if (fork_reduce) {
    // p == 1: C2b's partials reduced and the line search run by one kernel (its last CTA)
    OFSC_CUDA(cudaStreamWaitEvent(s, w.ev_f1, 0));
    // PDL edge from C2b (the joined Q/P reduction stays a full dependency)
    pdl_next(pdl && pdl_ls());
    pr.ph(OFSC_PH_LINE_SEARCH, 1, [&] {
      if (diag) launch_reduce_linesearch(p, w.part_gd, w.nbd, 1, s);
      else launch_reduce_linesearch(p, w.part_g2, w.nb2, 0, s);
    });
    return;
  }
  pr.ph(OFSC_PH_GRAM_REDUCE, 2, [&] {
    launch_reduce_partials(w.part_g4, w.nb4, 2 * p.KP * p.KP, w.grams, s);
    if (diag) {
      launch_reduce_partials(w.part_gd, w.nbd, 2 * p.KP, p.diagred, s);
      launch_expand_diag(p, s);
    } else {
      launch_reduce_partials(w.part_g2, w.nb2, 2 * p.KP * p.KP, w.grams + 2 * p.KP * p.KP, s);
    }
  });
  pr.ph(OFSC_PH_COMM, 0, [&] { allreduce_d(g, w.grams, 4 * (size_t)p.KP * p.KP, s); });
  pr.ph(OFSC_PH_LINE_SEARCH, 1, [&] { launch_linesearch(p, s); });
}

static bool use_graphs(ofsc_graph g) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("OFSC_NO_GRAPH");
    env = (e && e[0] == '1') ? 0 : 1;
  }
  // p > 1: captured with the NCCL calls inside (the init refresh before the capture
  // has already connected every peer); the local world's host barriers cannot be captured
  return env == 1 && (g->p == 1 || (g->comm && g->comm->nccl));
}

// Device-side iteration loop: a CUDA graph whose single node is a conditional
// WHILE node; its body is one captured iteration followed by k_loop_cond, which
// sets the condition from the control block (no host round trip per iteration,
// also in tolerance mode).  Opt-in (OFSC_DEVLOOP=1) for tolerance-mode runs:
// measured (tools/tol_loop_ab.py) 3x faster than host polling on c1 (80 vs 250
// us/iteration) but ~20 % slower on c2 and neutral on c3, where the while
// node's per-iteration body relaunch costs more than the host's queued launches.
__global__ void k_loop_cond(const DevCtl* ctl, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (ctl->stop == 0 && ctl->iter < ctl->limit) ? 1u : 0u);
}

static bool use_devloop() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("OFSC_DEVLOOP");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  return env == 1;
}

static void capture_loop(cudaGraph_t* gr, cudaGraphExec_t* ex, cudaStream_t s, const DevCtl* ctl,
                         const std::function<void()>& body) {
  OFSC_CUDA(cudaGraphCreate(gr, 0));
  cudaGraphConditionalHandle h;
  OFSC_CUDA(cudaGraphConditionalHandleCreate(&h, *gr, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  OFSC_CUDA(cudaGraphAddNode(&node, *gr, nullptr, 0, &np));
  cudaGraph_t bodyg = np.conditional.phGraph_out[0];
  OFSC_CUDA(cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
  try {
    body();
    k_loop_cond<<<1, 1, 0, s>>>(ctl, h);
    OFSC_LAUNCH_CHECK();
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(s, &junk);
    throw;
  }
  cudaGraph_t out = nullptr;
  OFSC_CUDA(cudaStreamEndCapture(s, &out));
  OFSC_CUDA(cudaGraphInstantiate(ex, *gr, 0));
}

static void capture(cudaGraph_t* gr, cudaGraphExec_t* ex, cudaStream_t s,
                    const std::function<void()>& body) {
  OFSC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(s, &junk);
    if (junk) cudaGraphDestroy(junk);
    throw;
  }
  OFSC_CUDA(cudaStreamEndCapture(s, gr));
  OFSC_CUDA(cudaGraphInstantiate(ex, *gr, 0));
}

}  // namespace ofsc

extern "C" {

ofsc_status ofsc_run_ex(ofsc_graph g, ofsc_method method, ofsc_dtype dt, const ofsc_opts* opts,
                        void* d_X, int64_t ldx, double* h_history, double* h_alphas,
                        int32_t* h_codes, ofsc_report* rep, ofsc_stream stream) {
  bool diverged = false;
  ofsc_status st = guard([&] {
    OFSC_REQUIRE(g && opts && d_X, OFSC_ERR_ARG, "null argument");
    const ofsc_opts o = *opts;
    OFSC_REQUIRE(method >= 0 && method <= 3, OFSC_ERR_ARG, "bad method");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    OFSC_REQUIRE(o.k >= 1 && o.k <= OFSC_MAX_K && o.k <= g->n, OFSC_ERR_ARG, "need 1 <= k <= min(n, 64)");
    OFSC_REQUIRE(ldx >= o.k && o.max_iters >= 0, OFSC_ERR_ARG, "bad ldx / max_iters");
    OFSC_REQUIRE(o.beta_rule >= 0 && o.beta_rule <= 2 && o.refresh >= 0 && o.tol >= 0.0,
                 OFSC_ERR_ARG, "bad options");
    OFSC_REQUIRE(g->p == 1 || comm_active(g->comm), OFSC_ERR_STATE,
                 "ofsc_run needs an NCCL communicator or a local world when p > 1 "
                 "(bare local test communicator given)");
    cudaStream_t s = (cudaStream_t)stream;
    const int KP = padded_k(o.k);
    trace_point("run: start", s);
    ensure_workspace(g, dt, KP, s);
    trace_point("run: workspace", s);
    Workspace& w = g->ws;
    const int T = o.max_iters;
    const size_t es = esize(dt);
    IterParams p = make_params(g, method, o, KP);
    DBuf hist((size_t)std::max(T, 1) * 4 * 8, s);
    DBuf halpha(h_alphas ? (size_t)std::max(T, 1) * KP * 8 : 0, s);
    DBuf hcode(h_codes ? (size_t)std::max(T, 1) * KP * 4 : 0, s);
    p.hist = hist.as<double>();
    p.hist_alpha = halpha.as<double>();
    p.hist_code = hcode.as<int>();
    OFSC_CUDA(cudaMemsetAsync(p.hist, 0xff, (size_t)std::max(T, 1) * 4 * 8, s));  // NaN
    const size_t blk = (size_t)std::max<int64_t>(g->n_local, 1) * KP * es;
    const size_t vg = g->p == 1 ? blk : (size_t)g->ext_rows * KP * es;
    launch_copy_in(dt, o.k, KP, g->n_local, d_X, ldx, w.X, g->user_perm(), s);
    OFSC_CUDA(cudaMemsetAsync(w.G, 0, blk, s));
    OFSC_CUDA(cudaMemsetAsync(w.AV, 0, blk, s));
    OFSC_CUDA(cudaMemsetAsync(w.Vg, 0, vg, s));
    OFSC_CUDA(cudaMemsetAsync(w.state, 0, (size_t)(2 * KP * KP + 7 * KP) * 8, s));
    OFSC_CUDA(cudaMemsetAsync(w.ctl, 0, sizeof(DevCtl), s));
    // init: AX = A X0, M = X0^T X0, W = X0^T A X0
    {
      Prof init;
      refresh_ops(g, dt, p, s, init);
    }
    trace_point("run: init refresh", s);
    // The iteration is captured once per call as CUDA graphs (plain and refresh
    // iteration); they bake in this call's history buffers.  Profiling runs
    // eager launches bracketed by events instead.
    bool graphs = use_graphs(g) && !o.profile;
    // device-side loop only on request and in tolerance mode; a fixed T launches the
    // captured iteration T times (measured faster: the host queues launches ahead)
    const bool devloop = graphs && g->p == 1 && o.refresh == 0 && o.tol > 0.0 && use_devloop();
    int n_launch_iter = 0, n_launch_refresh = 0;
    if (graphs) {
      if (w.e_iter) cudaGraphExecDestroy(w.e_iter);
      if (w.e_refresh) cudaGraphExecDestroy(w.e_refresh);
      if (w.e_loop) cudaGraphExecDestroy(w.e_loop);
      if (w.g_iter) cudaGraphDestroy(w.g_iter);
      if (w.g_refresh) cudaGraphDestroy(w.g_refresh);
      if (w.g_loop) cudaGraphDestroy(w.g_loop);
      w.e_iter = w.e_refresh = w.e_loop = nullptr;
      w.g_iter = w.g_refresh = w.g_loop = nullptr;
      // capture on a private stream (the caller's may be the legacy default stream,
      // which cannot be captured); the graphs are then launched on the caller's stream.
      if (!w.cap) OFSC_CUDA(cudaStreamCreateWithFlags(&w.cap, cudaStreamNonBlocking));
      Prof c1, c2;
      try {
        if (devloop) {
          capture_loop(&w.g_loop, &w.e_loop, w.cap, w.ctl,
                       [&] { iteration_ops(g, dt, p, false, w.cap, c1); });
          n_launch_iter = c1.total() + 1;   // + the loop-condition kernel
        } else {
          capture(&w.g_iter, &w.e_iter, w.cap, [&] { iteration_ops(g, dt, p, false, w.cap, c1); });
          n_launch_iter = c1.total();
        }
        if (o.refresh >= 1) {
          capture(&w.g_refresh, &w.e_refresh, w.cap,
                  [&] { iteration_ops(g, dt, p, true, w.cap, c2); });
          n_launch_refresh = c2.total();
        }
      } catch (const Error& e) {
        // p > 1: an NCCL build that cannot capture its calls -> eager launches
        // (same kernels and collectives, same arithmetic); p == 1 never falls back
        if (g->p == 1) throw;
        cudaGetLastError();
        if (w.e_iter) cudaGraphExecDestroy(w.e_iter);
        if (w.e_refresh) cudaGraphExecDestroy(w.e_refresh);
        if (w.g_iter) cudaGraphDestroy(w.g_iter);
        if (w.g_refresh) cudaGraphDestroy(w.g_refresh);
        w.e_iter = w.e_refresh = nullptr;
        w.g_iter = w.g_refresh = nullptr;
        graphs = false;
        if (getenv("OFSC_TRACE"))
          fprintf(stderr, "[ofsc] p > 1 iteration not captured (%s): eager launches\n",
                  e.msg.c_str());
      }
    }
    trace_point("run: graphs captured", s);
    int* h_stop = nullptr;
    OFSC_CUDA(cudaMallocHost(&h_stop, sizeof(int)));
    struct HostFree {
      int* q;
      ~HostFree() { cudaFreeHost(q); }
    } hf{h_stop};
    const int check = o.tol > 0.0 ? std::max(1, o.check_every) : 0;
    const int t0 = o.timing_skip >= 0 ? o.timing_skip : (o.profile ? 0 : T + 1);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    struct EvFree {
      cudaEvent_t* a;
      cudaEvent_t* b;
      ~EvFree() {
        if (*a) cudaEventDestroy(*a);
        if (*b) cudaEventDestroy(*b);
      }
    } evf{&ev0, &ev1};
    Prof prof, quiet;
    prof.timing = o.profile != 0;
    prof.s = s;
    int launches = 0, t_last = 0, timed_iters = 0;
    if (devloop) {
      // iterations [a, b) in one graph launch (the while node stops at b or at a stop flag)
      auto segment = [&](int a, int b) {
        if (b <= a) return;
        const int lim = b;
        OFSC_CUDA(cudaMemcpyAsync(&w.ctl->limit, &lim, sizeof(int), cudaMemcpyHostToDevice, s));
        OFSC_CUDA(cudaGraphLaunch(w.e_loop, s));
      };
      const int tw = std::min(std::max(t0, 0), T);
      segment(0, tw);
      if (t0 < T) {                                  // timing window [t0, T)
        OFSC_CUDA(cudaEventCreate(&ev0));
        OFSC_CUDA(cudaEventRecord(ev0, s));
      }
      segment(tw, T);
      DevCtl c0;
      OFSC_CUDA(cudaMemcpyAsync(&c0, w.ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, s));
      OFSC_CUDA(cudaStreamSynchronize(s));
      if (ev0) {
        timed_iters = std::max(0, std::min(c0.iter + (c0.stop ? 1 : 0), T) - tw);
        launches = timed_iters * n_launch_iter;
      }
      t_last = c0.iter;
    }
    for (int t = 0; t < T && !devloop; ++t) {
      const bool in_window = t >= t0;
      if (t == t0) {
        OFSC_CUDA(cudaEventCreate(&ev0));
        OFSC_CUDA(cudaEventRecord(ev0, s));
      }
      const bool refresh = t > 0 && o.refresh >= 1 && t % o.refresh == 0;
      if (graphs) {
        OFSC_CUDA(cudaGraphLaunch(refresh ? w.e_refresh : w.e_iter, s));
        if (in_window) launches += refresh ? n_launch_refresh : n_launch_iter;
      } else {
        Prof& pr = in_window ? prof : quiet;
        const int before = pr.total();
        iteration_ops(g, dt, p, refresh, s, pr);
        if (in_window) launches += pr.total() - before;
      }
      if (in_window) ++timed_iters;
      t_last = t + 1;
      if (check && (t + 1) % check == 0) {
        OFSC_CUDA(cudaMemcpyAsync(h_stop, &w.ctl->stop, sizeof(int), cudaMemcpyDeviceToHost, s));
        OFSC_CUDA(cudaStreamSynchronize(s));
        if (*h_stop) break;
      }
    }
    if (ev0) {
      OFSC_CUDA(cudaEventCreate(&ev1));
      OFSC_CUDA(cudaEventRecord(ev1, s));
    }
    (void)t_last;
    launch_update_x(dt, p, s);  // pending step of the last iteration (no-op after a stop)
    launch_copy_out(dt, o.k, KP, g->n_local, w.X, d_X, ldx, g->user_perm(), s);
    DevCtl c;
    OFSC_CUDA(cudaMemcpyAsync(&c, w.ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, s));
    std::vector<double> hh((size_t)std::max(T, 1) * 4);
    OFSC_CUDA(cudaMemcpyAsync(hh.data(), p.hist, hh.size() * 8, cudaMemcpyDeviceToHost, s));
    std::vector<double> ha;
    std::vector<int> hc;
    if (h_alphas) {
      ha.resize((size_t)std::max(T, 1) * KP);
      OFSC_CUDA(cudaMemcpyAsync(ha.data(), p.hist_alpha, ha.size() * 8, cudaMemcpyDeviceToHost, s));
    }
    if (h_codes) {
      hc.resize((size_t)std::max(T, 1) * KP);
      OFSC_CUDA(cudaMemcpyAsync(hc.data(), p.hist_code, hc.size() * 4, cudaMemcpyDeviceToHost, s));
    }
    OFSC_CUDA(cudaStreamSynchronize(s));
    if (h_history) std::memcpy(h_history, hh.data(), (size_t)T * 4 * 8);
    for (int t = 0; t < T; ++t)
      for (int j = 0; j < o.k; ++j) {
        const bool done = t < c.iter || (c.stop == 2 && t == c.iter);
        if (h_alphas) h_alphas[(size_t)t * o.k + j] = done ? ha[(size_t)t * KP + j] : NAN;
        if (h_codes) h_codes[(size_t)t * o.k + j] = done ? hc[(size_t)t * KP + j] : -1;
      }
    if (rep) {
      rep->iters = c.iter;
      rep->converged = c.stop == 1;
      rep->diverged = c.stop == 2;
      rep->n_three_root_steps = c.n_three;
      rep->n_zero_steps = c.n_zero;
      rep->grad_norm0 = c.gnorm0;
      rep->grad_norm = c.gnorm;
      rep->objective = c.obj;
      rep->timed_iters = timed_iters;
      rep->launches = launches;
      rep->timed_ms = 0.0;
      if (ev0 && ev1) {
        float ms = 0.f;
        OFSC_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
        rep->timed_ms = ms;
      }
      for (int q = 0; q < OFSC_NUM_PHASES; ++q) {
        rep->kernel_ms[q] = 0.0;
        rep->kernel_launches[q] = o.profile ? prof.launches[q] : 0;
      }
      if (o.profile) prof.resolve(rep->kernel_ms);
    }
    diverged = c.stop == 2;
  });
  if (st == OFSC_OK && diverged) {
    set_last_error("non-finite direction or step; X holds the last finite iterate");
    return OFSC_ERR_DIVERGED;
  }
  return st;
}

ofsc_status ofsc_run(ofsc_graph g, ofsc_method method, ofsc_dtype dt, const ofsc_opts* opts,
                     void* d_X, int64_t ldx, double* h_history, ofsc_report* rep,
                     ofsc_stream stream) {
  return ofsc_run_ex(g, method, dt, opts, d_X, ldx, h_history, nullptr, nullptr, rep, stream);
}

ofsc_status ofsc_line_search(ofsc_method method, int32_t k, const double* h_Q, const double* h_P,
                             const double* h_T, const double* h_Rp, const double* h_M,
                             const double* h_W, double* h_alpha, int32_t* h_codes,
                             double* h_M_out, double* h_W_out) {
  return guard([&] {
    OFSC_REQUIRE(h_Q && h_P && h_T && h_Rp && h_M && h_W && h_alpha && k >= 1 && k <= OFSC_MAX_K,
                 OFSC_ERR_ARG, "bad line-search args");
    OFSC_REQUIRE(method >= 0 && method <= 3, OFSC_ERR_ARG, "bad method");
    const int KP = padded_k(k);
    cudaStream_t s = nullptr;
    DBuf in((size_t)6 * k * k * 8, s), gr((size_t)6 * KP * KP * 8, s), al((size_t)KP * 8, s),
        cd((size_t)KP * 4, s);
    const double* src[6] = {h_Q, h_P, h_T, h_Rp, h_M, h_W};
    for (int q = 0; q < 6; ++q)
      OFSC_CUDA(cudaMemcpyAsync(in.as<double>() + q * k * k, src[q], (size_t)k * k * 8,
                                cudaMemcpyHostToDevice, s));
    for (int q = 0; q < 6; ++q)
      k_embed_kk<<<(KP * KP + 255) / 256, 256, 0, s>>>(in.as<double>() + q * k * k, KP, k,
                                                       gr.as<double>() + q * KP * KP);
    OFSC_LAUNCH_CHECK();
    double* M = gr.as<double>() + 4 * KP * KP;
    double* W = gr.as<double>() + 5 * KP * KP;
    launch_linesearch_hook(method, k, KP, gr.as<double>(), M, W, al.as<double>(), cd.as<int>(), s);
    std::vector<double> a(KP), mw(2 * KP * KP);
    std::vector<int> c(KP);
    OFSC_CUDA(cudaMemcpyAsync(a.data(), al.p, KP * 8, cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaMemcpyAsync(c.data(), cd.p, KP * 4, cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaMemcpyAsync(mw.data(), M, 2 * KP * KP * 8, cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < k; ++i) {
      h_alpha[i] = a[i];
      if (h_codes) h_codes[i] = c[i];
      for (int j = 0; j < k; ++j) {
        if (h_M_out) h_M_out[i * k + j] = mw[i * KP + j];
        if (h_W_out) h_W_out[i * k + j] = mw[KP * KP + i * KP + j];
      }
    }
  });
}

// ---------------------------------------------------------------------------
// post-processing
// ---------------------------------------------------------------------------
ofsc_status ofsc_row_normalize(ofsc_dtype dt, int64_t n_local, int32_t k, const void* d_X,
                               int64_t ldx, void* d_Y, int64_t ldy, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(d_X && d_Y && n_local >= 0 && k >= 1 && k <= OFSC_MAX_K && ldx >= k && ldy >= k,
                 OFSC_ERR_ARG, "bad normalize args");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    if (n_local == 0) return;
    launch_row_normalize(dt, n_local, k, d_X, ldx, d_Y, ldy, (cudaStream_t)stream);
  });
}

namespace ofsc {
// K-means step counters (changes, skipped, product blocks) and inertia -> mapped host memory
__global__ void k_publish_counters(const unsigned long long* chg, const double* tot,
                                   unsigned long long* h) {
  if (threadIdx.x < 3) ((volatile unsigned long long*)h)[threadIdx.x] = chg[threadIdx.x];
  if (threadIdx.x == 3) ((volatile unsigned long long*)h)[3] = __double_as_longlong(*tot);
  __threadfence_system();
}
}  // namespace ofsc

ofsc_status ofsc_kmeans(ofsc_comm comm, ofsc_dtype dt, int64_t n_local, int32_t dim,
                        const void* d_Y, int64_t ldy, int32_t n_clusters, double* d_centroids,
                        int32_t max_iters, int32_t* d_labels, int32_t* iters_out,
                        double* inertia_out, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(d_Y && d_centroids && d_labels && n_local >= 0 && dim >= 1 && ldy >= dim &&
                     n_clusters >= 1 && n_clusters <= 128 && max_iters >= 1,
                 OFSC_ERR_ARG, "bad kmeans args");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    OFSC_REQUIRE(!comm || comm->nranks == 1 || comm_active(comm), OFSC_ERR_STATE,
                 "ofsc_kmeans needs an NCCL communicator or a local world when p > 1");
    cudaStream_t s = (cudaStream_t)stream;
    const int K = n_clusters;
    const bool fused = kmeans_step_supported(dim, K);   // assign + partial sums in one pass
    const int nb = fused ? kmeans_step_blocks(std::max<int64_t>(n_local, 1))
                         : kmeans_blocks(std::max<int64_t>(n_local, 1));
    const int nbp = fused ? nb : kmeans_partial_blocks(std::max<int64_t>(n_local, 1));
    const int W = dim + 1;
    const int P = comm ? comm->nranks : 1;
    DBuf chg(3 * 8, s), pin((size_t)nb * 8, s), part((size_t)nbp * K * W * 8, s),
        red((size_t)K * W * 8, s), tot(8, s),
        gat(P > 1 ? (size_t)P * std::max(K * W, 3) * 8 : 0, s),
        lbd(fused ? (size_t)std::max<int64_t>(n_local, 1) * 8 : 8, s), dlt((size_t)K * 8, s),
        sep((size_t)K * 8, s);
    // light steps (bounds first, sums by label changes; kernels_kmeans.cu): once at
    // most 1/8 of the rows failed the previous step's bound tests (the light step
    // assigns those by the direct form, without tensor cores).  S = running sums.
    const bool light_ok = fused && kmeans_light_supported(dim, K);
    const int nbl = light_ok ? kmeans_light_blocks(std::max<int64_t>(n_local, 1)) : 0;
    DBuf ubd(light_ok ? (size_t)std::max<int64_t>(n_local, 1) * 8 : 8, s),
        Ssum((size_t)K * W * 8, s), partl(light_ok ? (size_t)nbl * K * W * 8 : 8, s);
    unsigned long long n_total = (unsigned long long)std::max<int64_t>(n_local, 0);
    if (light_ok && comm_active(comm)) {
      DBuf nt(8, s);
      OFSC_CUDA(cudaMemcpyAsync(nt.p, &n_total, 8, cudaMemcpyHostToDevice, s));
      comm_sum_u64(comm, nt.as<unsigned long long>(), 1, gat.as<unsigned long long>(), s);
      OFSC_CUDA(cudaMemcpyAsync(&n_total, nt.p, 8, cudaMemcpyDeviceToHost, s));
      OFSC_CUDA(cudaStreamSynchronize(s));
    }
    unsigned long long prev_fail = ~0ull;
    OFSC_CUDA(cudaMemsetAsync(d_labels, 0xff, std::max<int64_t>(n_local, 0) * sizeof(int32_t), s));
    // pinned counter readback, allocated once per host thread (cudaFreeHost would
    // synchronise the whole device, e.g. the feature download of spectral_cluster)
    // published by a kernel into mapped host memory: no copy-engine transfer, so the
    // per-step readback never queues behind a large download (spectral_cluster's
    // features overlap K-means on a side stream)
    static thread_local unsigned long long* h_chg = nullptr;
    static thread_local unsigned long long* d_hchg = nullptr;
    if (!h_chg) {
      OFSC_CUDA(cudaHostAlloc((void**)&h_chg, 4 * 8, cudaHostAllocMapped));
      OFSC_CUDA(cudaHostGetDevicePointer((void**)&d_hchg, h_chg, 0));
    }
    const bool stats = getenv("OFSC_KMEANS_STATS") != nullptr;   // per-step skip statistics
    const bool noskip = getenv("OFSC_KMEANS_NOSKIP") != nullptr; // A/B: no bound test
    const char* elk = getenv("OFSC_KMEANS_ELKAN");                // A/B: 0 = Hamerly bound only
    const bool elkan = !(elk && elk[0] == '0');
    int it = 0;
    double inertia = 0.0;
    for (it = 1; it <= max_iters; ++it) {
      OFSC_CUDA(cudaMemsetAsync(chg.p, 0, 3 * 8, s));
      OFSC_CUDA(cudaMemsetAsync(pin.p, 0, (size_t)nb * 8, s));
      cudaEvent_t ea = nullptr, eb = nullptr;
      if (stats) {
        OFSC_CUDA(cudaEventCreate(&ea));
        OFSC_CUDA(cudaEventCreate(&eb));
        OFSC_CUDA(cudaEventRecord(ea, s));
      }
      const bool light = light_ok && it > 1 && !noskip && elkan && prev_fail * 8 <= n_total;
      if (n_local > 0 && light)
        launch_kmeans_light(dt, n_local, dim, d_Y, ldy, K, d_centroids, d_labels, ubd.as<double>(),
                            lbd.as<double>(), dlt.as<double>(), sep.as<double>(),
                            chg.as<unsigned long long>(), partl.as<double>(), nbl, s);
      else if (n_local > 0 && fused)
        launch_kmeans_step(dt, n_local, dim, d_Y, ldy, K, d_centroids, d_labels,
                           chg.as<unsigned long long>(), pin.as<double>(), part.as<double>(),
                           lbd.as<double>(), it > 1 && !noskip ? dlt.as<double>() : nullptr,
                           elkan ? sep.as<double>() : nullptr,
                           light_ok ? ubd.as<double>() : nullptr, nb, s);
      else if (n_local > 0)
        launch_kmeans_assign(dt, n_local, dim, d_Y, ldy, K, d_centroids, d_labels,
                             chg.as<unsigned long long>(), pin.as<double>(), nb, s);
      if (stats) OFSC_CUDA(cudaEventRecord(eb, s));
      launch_reduce_partials(pin.as<double>(), nb, 1, tot.as<double>(), s);
      if (comm_active(comm)) {
        comm_sum_u64(comm, chg.as<unsigned long long>(), 3, gat.as<unsigned long long>(), s);
        comm_sum_f64(comm, tot.as<double>(), 1, gat.as<double>(), s);
      }
      k_publish_counters<<<1, 32, 0, s>>>(chg.as<unsigned long long>(), tot.as<double>(), d_hchg);
      OFSC_LAUNCH_CHECK();
      OFSC_CUDA(cudaStreamSynchronize(s));
      if (stats) {
        float ms = 0.f;
        OFSC_CUDA(cudaEventElapsedTime(&ms, ea, eb));
        cudaEventDestroy(ea);
        cudaEventDestroy(eb);
        fprintf(stderr, "[ofsc kmeans] step %d changes %llu skipped %llu product_blocks %llu ms %.3f light %d\n",
                it, h_chg[0], h_chg[1], h_chg[2], ms, light ? 1 : 0);
      }
      {
        double v;
        memcpy(&v, (const void*)&((volatile unsigned long long*)h_chg)[3], 8);
        inertia = v;
      }
      const unsigned long long nchanged = ((volatile unsigned long long*)h_chg)[0];
      const bool last = (it > 1 && nchanged == 0) || it == max_iters;
      if (light && last) {
        // the light step does not visit every row: the inertia of this (final)
        // assignment comes from one pass with the centroids it used
        if (n_local > 0)
          launch_kmeans_inertia(dt, n_local, dim, d_Y, ldy, d_centroids, d_labels, pin.as<double>(),
                                nb, s);
        launch_reduce_partials(pin.as<double>(), nb, 1, tot.as<double>(), s);
        if (comm_active(comm)) comm_sum_f64(comm, tot.as<double>(), 1, gat.as<double>(), s);
        OFSC_CUDA(cudaMemcpyAsync(&inertia, tot.p, 8, cudaMemcpyDeviceToHost, s));
        OFSC_CUDA(cudaStreamSynchronize(s));
      }
      {
        const unsigned long long nsk = ((volatile unsigned long long*)h_chg)[1];
        prev_fail = n_total > nsk ? n_total - nsk : 0;
      }
      if (it > 1 && nchanged == 0) break;
      if (light) {
        if (n_local == 0) OFSC_CUDA(cudaMemsetAsync(partl.p, 0, (size_t)nbl * K * W * 8, s));
        launch_reduce_partials(partl.as<double>(), nbl, K * W, red.as<double>(), s);
        if (comm_active(comm)) comm_sum_f64(comm, red.as<double>(), (size_t)K * W, gat.as<double>(), s);
        launch_kmeans_accum(K * W, Ssum.as<double>(), red.as<double>(), s);
      } else {
        if (n_local > 0 && !fused)
          launch_kmeans_partial(dt, n_local, dim, d_Y, ldy, K, d_labels, part.as<double>(), nbp, s);
        else if (n_local == 0)
          OFSC_CUDA(cudaMemsetAsync(part.p, 0, (size_t)nbp * K * W * 8, s));
        launch_reduce_partials(part.as<double>(), nbp, K * W, Ssum.as<double>(), s);
        if (comm_active(comm)) comm_sum_f64(comm, Ssum.as<double>(), (size_t)K * W, gat.as<double>(), s);
      }
      if (fused) {
        launch_kmeans_finish_delta(K, dim, Ssum.as<double>(), d_centroids, dlt.as<double>(), s);
        launch_kmeans_halfsep(K, dim, d_centroids, sep.as<double>(), s);
      }
      else launch_kmeans_finish(K, dim, Ssum.as<double>(), d_centroids, s);
    }
    OFSC_CUDA(cudaStreamSynchronize(s));
    if (iters_out) *iters_out = std::min(it, max_iters);
    if (inertia_out) *inertia_out = inertia;
  });
}

ofsc_status ofsc_rayleigh_ritz(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_X,
                               int64_t ldx, void* d_U, int64_t ldu, double* h_theta,
                               double* h_relerr, ofsc_stream stream) {
  return guard([&] {
    OFSC_REQUIRE(g && d_X && h_theta, OFSC_ERR_ARG, "null argument");
    OFSC_REQUIRE(dt == OFSC_F64 || dt == OFSC_F32, OFSC_ERR_ARG, "bad dtype");
    OFSC_REQUIRE(k >= 1 && k <= OFSC_MAX_K && k <= g->n, OFSC_ERR_ARG,
                 "need 1 <= k <= min(n, 64)");
    OFSC_REQUIRE(ldx >= k && (!d_U || ldu >= k), OFSC_ERR_ARG, "bad ldx / ldu");
    OFSC_REQUIRE(g->p == 1 || comm_active(g->comm), OFSC_ERR_STATE,
                 "ofsc_rayleigh_ritz needs an NCCL communicator or a local world when p > 1");
    cudaStream_t s = (cudaStream_t)stream;
    const int KP = padded_k(k);
    ensure_workspace(g, dt, KP, s);
    Workspace& w = g->ws;
    ofsc_opts o{};
    o.k = k;
    IterParams p = make_params(g, OFSC_OFM_F2, o, KP);
    launch_copy_in(dt, k, KP, g->n_local, d_X, ldx, w.X, g->user_perm(), s);
    OFSC_CUDA(cudaMemsetAsync(w.ctl, 0, sizeof(DevCtl), s));
    {
      Prof pr;
      refresh_ops(g, dt, p, s, pr);   // A X, M = X^T X, W = X^T A X (reduced over ranks)
    }
    const int nb = rr_rows_blocks(std::max<int64_t>(g->n_local, 1));
    DBuf tm((size_t)KP * KP * 8, s), th((size_t)KP * 8, s), stt(8, s), part((size_t)nb * 2 * 8, s),
        red(2 * 8, s);
    launch_rr_small(p.M, p.W, KP, k, tm.as<double>(), th.as<double>(), stt.as<int>(), s);
    int bad = 0;
    OFSC_CUDA(cudaMemcpyAsync(&bad, stt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaStreamSynchronize(s));
    OFSC_REQUIRE(!bad, OFSC_ERR_RANGE, "X^T X is not positive definite (X rank deficient)");
    if (g->n_local > 0)
      launch_rr_rows(dt, g->n_local, k, KP, w.X, w.AX, tm.as<double>(), th.as<double>(), w.G,
                     part.as<double>(), nb, s);
    else
      OFSC_CUDA(cudaMemsetAsync(part.p, 0, (size_t)nb * 2 * 8, s));
    launch_reduce_partials(part.as<double>(), nb, 2, red.as<double>(), s);
    allreduce_d(g, red.as<double>(), 2, s);
    if (d_U) launch_copy_out(dt, k, KP, g->n_local, w.G, d_U, ldu, g->user_perm(), s);
    double hr[2];
    std::vector<double> ht(KP);
    OFSC_CUDA(cudaMemcpyAsync(hr, red.p, 2 * 8, cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaMemcpyAsync(ht.data(), th.p, (size_t)KP * 8, cudaMemcpyDeviceToHost, s));
    OFSC_CUDA(cudaStreamSynchronize(s));
    for (int j = 0; j < k; ++j) h_theta[j] = ht[j];
    if (h_relerr) *h_relerr = hr[1] > 0.0 ? std::sqrt(hr[0]) / std::sqrt(hr[1]) : 0.0;
  });
}

ofsc_status ofsc_scores(int64_t n, const int32_t* a, const int32_t* b, double* ari, double* nmi) {
  return guard([&] {
    OFSC_REQUIRE(a && b && n >= 1, OFSC_ERR_ARG, "bad scores args");
    std::map<int32_t, int> ia, ib;
    for (int64_t i = 0; i < n; ++i) {
      ia.emplace(a[i], (int)ia.size());
      ib.emplace(b[i], (int)ib.size());
    }
    const size_t ra = ia.size(), rb = ib.size();
    std::vector<int64_t> C(ra * rb, 0), sa(ra, 0), sb(rb, 0);
    for (int64_t i = 0; i < n; ++i) {
      const int x = ia[a[i]], y = ib[b[i]];
      ++C[(size_t)x * rb + y];
      ++sa[x];
      ++sb[y];
    }
    auto c2 = [](double x) { return x * (x - 1.0) / 2.0; };
    double sij = 0, sA = 0, sB = 0;
    for (int64_t v : C) sij += c2((double)v);
    for (int64_t v : sa) sA += c2((double)v);
    for (int64_t v : sb) sB += c2((double)v);
    const double e = n > 1 ? sA * sB / c2((double)n) : 0.0;
    const double den = 0.5 * (sA + sB) - e;
    if (ari) *ari = den == 0.0 ? 1.0 : (sij - e) / den;
    if (nmi) {
      double ha = 0, hb = 0, mi = 0;
      const double N = (double)n;
      for (int64_t v : sa)
        if (v) ha -= (v / N) * std::log(v / N);
      for (int64_t v : sb)
        if (v) hb -= (v / N) * std::log(v / N);
      for (size_t x = 0; x < ra; ++x)
        for (size_t y = 0; y < rb; ++y) {
          const int64_t v = C[x * rb + y];
          if (v) mi += (v / N) * std::log((v / N) / ((sa[x] / N) * (sb[y] / N)));
        }
      *nmi = (ha + hb == 0.0) ? 1.0 : 2.0 * mi / (ha + hb);
    }
  });
}

}  // extern "C"

namespace ofsc {
// C[c] = Y[local row of node init_rows[c]] if this rank owns it, else 0 (summed over ranks)
__global__ void k_gather_rows(int K, int dim, const int64_t* rows, const int32_t* inv,
                              int64_t row_begin, int64_t n_local, const void* Y, int64_t ldy,
                              int f64, double* C) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K * dim) return;
  const int c = e / dim, d = e % dim;
  const int64_t node = rows[c];
  const int64_t r = (inv ? (int64_t)inv[node] : node) - row_begin;
  double v = 0.0;
  if (r >= 0 && r < n_local)
    v = f64 ? ((const double*)Y)[r * ldy + d] : (double)((const float*)Y)[r * ldy + d];
  C[e] = v;
}
__global__ void k_invert_perm(int64_t n, const int32_t* perm, int32_t* inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}
// local internal rows <-> rows of a full original-order array
__global__ void k_scatter_labels(int64_t n_local, int64_t row_begin, const int32_t* perm,
                                 const int32_t* lab, int32_t* full) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_local;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = row_begin + i;
    full[perm ? perm[g] : g] = lab[i];
  }
}
}  // namespace ofsc

extern "C" ofsc_status ofsc_spectral_cluster(ofsc_comm comm, int64_t n, int64_t m,
                                             const int64_t* h_src, const int64_t* h_dst,
                                             ofsc_method method, ofsc_dtype dt,
                                             const ofsc_opts* opts, const ofsc_build_opts* bopts,
                                             void* h_X, int32_t n_clusters,
                                             const int64_t* h_init_rows, int32_t km_max_iters,
                                             int32_t* h_labels, ofsc_report* rep,
                                             ofsc_stream stream) {
  ofsc_graph g = nullptr;
  ofsc_status run_st = OFSC_OK;
  ofsc_status st = guard([&] {
    OFSC_REQUIRE(opts && h_X && h_init_rows && h_labels && n_clusters >= 1 && opts->k >= 1,
                 OFSC_ERR_ARG, "bad spectral_cluster args");
    cudaStream_t s = (cudaStream_t)stream;
    trace_point("spectral_cluster: enter", s);
    // copies overlap compute on a side stream: X0 upload || graph build,
    // feature download || normalise + K-means (pinned host buffers make them async)
    // (declared after dXf: destroyed first, so the side stream is drained before
    // dXf is released on `s`, also on error paths)
    const int k = opts->k;
    const size_t es = esize(dt);
    DBuf dXf((size_t)n * k * es, s);
    struct Side {
      cudaStream_t st = nullptr;
      cudaEvent_t a = nullptr, b = nullptr;
      ~Side() {
        if (st) cudaStreamSynchronize(st);
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        if (st) cudaStreamDestroy(st);
      }
    } side;
    OFSC_CUDA(cudaStreamCreateWithFlags(&side.st, cudaStreamNonBlocking));
    OFSC_CUDA(cudaEventCreateWithFlags(&side.a, cudaEventDisableTiming));
    OFSC_CUDA(cudaEventCreateWithFlags(&side.b, cudaEventDisableTiming));
    // the edges go first (the build needs them), X0 follows on the side stream
    // while the graph is built (the run needs it only after the build)
    DBuf de(m > 0 ? (size_t)m * 2 * sizeof(int64_t) : 0, s);
    if (m > 0) {
      OFSC_CUDA(cudaMemcpyAsync(de.p, h_src, (size_t)m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      OFSC_CUDA(cudaMemcpyAsync(de.as<int64_t>() + m, h_dst, (size_t)m * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
    }
    OFSC_CUDA(cudaEventRecord(side.b, s));                 // dXf allocated, edges uploaded
    OFSC_CUDA(cudaStreamWaitEvent(side.st, side.b, 0));
    OFSC_CUDA(cudaMemcpyAsync(dXf.p, h_X, (size_t)n * k * es, cudaMemcpyHostToDevice, side.st));
    OFSC_CUDA(cudaEventRecord(side.a, side.st));
    trace_point("spectral_cluster: X0 uploaded (side stream)", side.st);
    // default: reorder when the run is long enough to repay the LPA pass
    // (c4: ~60 ms for LPA + second CSR build vs ~3 ms saved per iteration;
    // profiles/r01/SUMMARY.md, tools/build_probe.py)
    ofsc_build_opts bo{opts->max_iters >= 32 ? 1 : 0, 30};
    if (bopts) bo = *bopts;
    trace_point("spectral_cluster: start", s);
    ofsc_status b = ofsc_graph_build_ex(comm, n, m, m > 0 ? de.as<int64_t>() : h_src,
                                        m > 0 ? de.as<int64_t>() + m : h_dst, m > 0 ? 1 : 0, &bo,
                                        stream, &g);
    de.release();
    if (b != OFSC_OK) throw Error{b, g_last_error};
    trace_point("spectral_cluster: graph built", s);
    const int64_t nl = g->n_local;
    const int32_t* perm = g->reordered ? g->perm : nullptr;
    DBuf dX(g->p > 1 ? (size_t)std::max<int64_t>(nl, 1) * k * es : 0, s),
        dY(std::max<int64_t>(nl, 1) * k * es, s), dC((size_t)n_clusters * k * 8, s),
        dL(std::max<int64_t>(nl, 1) * 4, s), dLf((size_t)n * 4, s), dR((size_t)n_clusters * 8, s),
        dInv(perm ? (size_t)n * 4 : 0, s);
    // all n rows of X0 (original order) -> this rank's internal rows
    OFSC_CUDA(cudaStreamWaitEvent(s, side.a, 0));
    // p == 1: ofsc_run maps original-order rows through perm itself, run on the full
    // array; p > 1: gather this rank's internal rows first
    void* Xrun = dXf.p;
    if (g->p > 1) {
      launch_copy_in(dt, k, k, nl,
                     (const char*)dXf.p + (perm ? 0 : (size_t)g->row_begin * k * es), k, dX.p,
                     perm ? perm + g->row_begin : nullptr, s);
      Xrun = dX.p;
    }
    trace_point("spectral_cluster: X0 on device", s);
    run_st = ofsc_run(g, method, dt, opts, Xrun, k, nullptr, rep, stream);
    trace_point("spectral_cluster: run done", s);
    if (run_st != OFSC_OK && run_st != OFSC_ERR_DIVERGED) throw Error{run_st, g_last_error};
    // features back to the caller's full array (rows this rank owns)
    if (g->p == 1) {
      OFSC_CUDA(cudaEventRecord(side.b, s));
      OFSC_CUDA(cudaStreamWaitEvent(side.st, side.b, 0));
      OFSC_CUDA(cudaMemcpyAsync(h_X, dXf.p, (size_t)n * k * es, cudaMemcpyDeviceToHost, side.st));
      trace_point("spectral_cluster: features downloaded (side stream)", side.st);
    } else {
      launch_copy_out(dt, k, k, nl, dX.p,
                      (char*)dXf.p + (perm ? 0 : (size_t)g->row_begin * k * es), k,
                      perm ? perm + g->row_begin : nullptr, s);
      OFSC_CUDA(cudaMemcpyAsync(h_X, dXf.p, (size_t)n * k * es, cudaMemcpyDeviceToHost, s));
    }
    ofsc_status r = ofsc_row_normalize(dt, nl, k, Xrun, k, dY.p, k, stream);
    if (r != OFSC_OK) throw Error{r, g_last_error};
    OFSC_CUDA(cudaMemcpyAsync(dR.p, h_init_rows, (size_t)n_clusters * 8, cudaMemcpyHostToDevice, s));
    // K-means rows: p == 1 holds original order (no inverse needed); p > 1 internal order
    const int32_t* inv = nullptr;
    if (perm && g->p > 1) {
      k_invert_perm<<<num_sms() * 8, 256, 0, s>>>(n, perm, dInv.as<int32_t>());
      OFSC_LAUNCH_CHECK();
      inv = dInv.as<int32_t>();
    }
    k_gather_rows<<<(n_clusters * k + 255) / 256, 256, 0, s>>>(
        n_clusters, k, dR.as<int64_t>(), inv, g->p == 1 ? 0 : g->row_begin, nl, dY.p, k,
        dt == OFSC_F64, dC.as<double>());
    OFSC_LAUNCH_CHECK();
    if (comm_active(comm)) {
      DBuf gat((size_t)comm->nranks * n_clusters * k * 8, s);
      comm_sum_f64(comm, dC.as<double>(), (size_t)n_clusters * k, gat.as<double>(), s);
    }
    trace_point("spectral_cluster: normalised", s);
    r = ofsc_kmeans(comm, dt, nl, k, dY.p, k, n_clusters, dC.as<double>(), km_max_iters,
                    dL.as<int32_t>(), nullptr, nullptr, stream);
    trace_point("spectral_cluster: kmeans done", s);
    if (r != OFSC_OK) throw Error{r, g_last_error};
    if (g->p == 1) {
      OFSC_CUDA(cudaMemcpyAsync(h_labels, dL.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    } else {
      OFSC_CUDA(cudaMemsetAsync(dLf.p, 0xff, (size_t)n * 4, s));
      k_scatter_labels<<<num_sms() * 8, 256, 0, s>>>(nl, g->row_begin, perm, dL.as<int32_t>(),
                                                    dLf.as<int32_t>());
      OFSC_LAUNCH_CHECK();
      std::vector<int32_t> tmp(n);
      OFSC_CUDA(cudaMemcpyAsync(tmp.data(), dLf.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
      OFSC_CUDA(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < n; ++i)
        if (tmp[i] >= 0) h_labels[i] = tmp[i];
    }
    trace_point("spectral_cluster: labels queued", s);
    OFSC_CUDA(cudaStreamSynchronize(side.st));
    trace_point("spectral_cluster: features downloaded", s);
    OFSC_CUDA(cudaStreamSynchronize(s));
  });
  if (g) ofsc_graph_destroy(g);
  trace_point("spectral_cluster: end", (cudaStream_t)stream);
  if (st == OFSC_OK && run_st == OFSC_ERR_DIVERGED) return OFSC_ERR_DIVERGED;
  return st;
}

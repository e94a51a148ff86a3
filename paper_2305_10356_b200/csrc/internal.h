// Internal declarations shared by the libofsc translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <climits>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ofsc.h"

namespace ofsc {

// ---- error plumbing: internal code throws, every ABI entry point catches ----
struct Error {
  ofsc_status st;
  std::string msg;
};
void set_last_error(const std::string& m);

#define OFSC_CUDA(x)                                                                    \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw ::ofsc::Error{OFSC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define OFSC_NCCL(x)                                                                    \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      throw ::ofsc::Error{OFSC_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)}; \
  } while (0)
#define OFSC_REQUIRE(cond, code, m)                       \
  do {                                                    \
    if (!(cond)) throw ::ofsc::Error{code, std::string(m)}; \
  } while (0)
#define OFSC_LAUNCH_CHECK() OFSC_CUDA(cudaGetLastError())

constexpr int kTR = 32;        // rows per tile of the row-wise kernels
constexpr int kThreads = 256;  // threads per CTA of the tiled kernels

// Padded feature width used on the device (columns k..KP-1 are kept at zero).
inline int padded_k(int k) { return k <= 16 ? 16 : k <= 32 ? 32 : k <= 48 ? 48 : 64; }

// Device control block of one run (stream-ordered, no host round trip).
struct DevCtl {
  int iter;      // completed updates of X
  int stop;      // 0 running, 1 converged, 2 diverged
  int n_three;   // line searches that chose among three real roots
  int n_zero;    // degenerate cubics
  double gnorm0, gnorm, obj;
  int limit;     // device-side loop (CUDA graph while node): run while iter < limit && !stop
  unsigned int ls_done;   // CTAs of k_reduce_linesearch done (the last one runs the line search)
};

// Everything the per-iteration kernels need, passed by value.
struct IterParams {
  int64_t n_local;      // rows owned by this rank
  int64_t own_off;      // slot id of local row 0 inside the gathered layout
  int k, KP, method, beta_rule, line_search, T;
  double alpha_fixed, tol, cm, fro2;
  // N x KP blocks (type set by the dtype of the run)
  void* X;
  void* AX;
  void* G;
  void* V;              // local rows of V (a view into Vg when p > 1)
  void* AV;
  const void* Vg;       // V for the gathers (all slots)
  // CSR
  const int64_t* row_ptr;
  const int32_t* col;   // slot ids
  const double* s;      // per slot id
  const float* s32;
  // k x k state (KP x KP, row-major, fp64)
  double* M;
  double* W;
  double* alpha;        // [KP]
  double* beta;         // [KP]
  double* gg_prev;      // [KP]
  double* colred;       // [2 KP] reduced (gg, dg) when p > 1
  double* grams;        // [4 KP KP]: Q, P, T, R'
  double* part_cols;    // [nblk][2][KP]
  double* part_g4;      // [nblk][2][KP][KP] (Q, P)
  double* part_g2;      // [nblk][2][KP][KP] (T, R')
  double* part_gd;      // [nblk][2][KP] column dots diag T, diag R' (f1 methods)
  double* diagred;      // [2 KP] their reduction
  DevCtl* ctl;
  unsigned long long* spmm_ctr;  // [4] SpMM row counters, zeroed by k_beta (PDL chain: no memset)
  double* hist;         // [T][4]
  double* hist_alpha;   // [T][KP]
  int* hist_code;       // [T][KP]
};

// ---- launchers (kernels_*.cu) ----
// Programmatic dependent launch for the NEXT kernel launched by this host thread
// (set by the iteration schedule before a launcher call; consumed by that call's
// first kernel launch).  OFSC_PDL=0 disables it.
void pdl_next(bool on);
bool pdl_take();
int grid_rows(int64_t n_rows, int blocks_per_sm);
int num_sms();
void keep_pool();    // default mempool keeps freed scratch (no per-build re-mapping)
// Every long-lived device buffer comes from the device's stream-ordered pool (kept
// mapped by keep_pool): freeing a multi-GB workspace then costs no unmapping and no
// device-wide synchronisation.  dev_free releases on the legacy stream: callers
// guarantee that no queued work still uses the buffer.
void dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p);                          // no queued work uses p any more
void dev_free_async(void* p, cudaStream_t st);   // stream-ordered on st
void dev_trim();   // release cached blocks and trim the pool of the current device
void trace_point(const char* what, cudaStream_t st);   // OFSC_TRACE=1: phase timestamps

// grid sizes of the TMA-pipelined streaming kernels (<= 4 * #SMs)
int c3_grid(ofsc_dtype dt, int KP, int method, int64_t n);
int c4_grid(ofsc_dtype dt, int KP, int64_t n);
// C3: X += alpha V, AX += alpha AV (if apply_update), G = g_m(X, AX, M, W), column partials.
void launch_update_direction(ofsc_dtype dt, const IterParams& p, int apply_update, int nblk,
                             cudaStream_t s);
// X += alpha V only (refresh iterations, final update); also used to write X out.
void launch_update_x(ofsc_dtype dt, const IterParams& p, cudaStream_t s);
// C4: V = -G + beta Vp, partial Grams Q = V^T V, P = V^T X.
void launch_direction_gram(ofsc_dtype dt, const IterParams& p, int nblk, cudaStream_t s);
struct HeavyRows;
// C2: Y = A Z (Z gathered; C2a), then the partial Grams over the own rows (C2b, a
// separate TMA-streamed DMMA kernel). mode 0: (Zown^T Y, Xown^T Y); mode 1: (Zown^T Zown, Zown^T Y)
struct SvalStream;
void launch_spmm_then_gram(ofsc_dtype dt, int KP, int64_t n_local, int64_t own_off,
                      const int64_t* row_ptr, const int32_t* col, const double* s,
                      const float* s32, const void* Zg, const void* Xown, void* Y,
                      double* part, int mode, const int* stop, int nblk, cudaStream_t st,
                      const HeavyRows* heavy = nullptr,
                      unsigned long long* ctr = nullptr,   // in-order row hand-out (L2 window)
                      const SvalStream* svs = nullptr,     // neighbour-scale stream (p == 1)
                      int64_t nnz = -1);
// C2a: Y = A Z only (KP-padded rows)
// cid/cstart (may be NULL): community of each row -> L2 evict_last for in-community
// neighbour rows, evict_first for the rest (p == 1 only)
// Degree-aware row binning (power-law rows): rows with more than `thresh`
// neighbours are skipped by the row-per-lane-group SpMM and split into chunks of
// <= kHeavyChunk neighbours processed in parallel; a finalize pass sums each
// heavy row's chunk partials in chunk order.
constexpr int64_t kHeavyThresh = 256;   // r22 (KP = 16): SpMM 21.4 ms unsplit, 4.5 at 4096, 3.1 at 256
constexpr int64_t kHeavyChunk = 512;
// Neighbour scales s_j for the SpMM of large graphs (p == 1), instead of a random
// 8-byte gather s[col[e]] per neighbour: mode 1 streams s_j per nonzero (sval[nnz]);
// mode 2 packs the column's node degree into the column stream (colpack[e] = col |
// deg << 23) and reads s_j from a per-degree table (sval[max_deg + 1]).
struct SvalStream {
  int mode = 0;
  double* sval = nullptr;
  float* sval32 = nullptr;
  int32_t* colpack = nullptr;
  void release();
};
struct HeavyRows {
  int64_t thresh = INT64_MAX;      // rows with deg > thresh are heavy
  int64_t n_rows = 0, n_chunks = 0;
  int32_t* rows = nullptr;         // [n_rows] heavy row ids
  int32_t* chunk_first = nullptr;  // [n_rows + 1] first chunk of each heavy row
  int64_t* chunk_beg = nullptr;    // [n_chunks] CSR offsets
  int64_t* chunk_end = nullptr;
  void* scratch = nullptr;         // [n_chunks][64] partial sums (double or float)
  void release();
};
void build_heavy(const int64_t* d_row_ptr, int64_t n_rows, HeavyRows& out, cudaStream_t st);
void launch_spmm(ofsc_dtype dt, int KP, int64_t n_local, int64_t own_off, const int64_t* row_ptr,
                 const int32_t* col, const double* s, const float* s32, const void* Zg, void* Y,
                 const int* stop, cudaStream_t st, const int32_t* cid = nullptr,
                 const int64_t* cstart = nullptr, unsigned long long* ctr = nullptr,
                 int phase = 0,    // 1: raw partial sums into Y; 2: continue from Y and finish
                 const HeavyRows* heavy = nullptr,
                 const SvalStream* svs = nullptr,   // neighbour-scale stream (p == 1), or NULL
                 int64_t nnz = -1);             // nonzeros of this CSR (L2-prefetch default), -1: unknown
void build_sval(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* s, const float* s32, int64_t max_deg, SvalStream& out,
                cudaStream_t st);
constexpr int kSpmmChunk = 8;  // rows per dynamic work grab of the SpMM
// C2b: TMA-streamed Gram pair over own rows (mode 0: Z^T Y, X^T Y; mode 1: Z^T Z, Z^T Y)
int gram_stream_grid(ofsc_dtype dt, int KP, int64_t n);
void launch_gram_stream(ofsc_dtype dt, int KP, int64_t n, const void* Zown, const void* Xown,
                        const void* Y, double* part, int mode, const int* stop, int nblk,
                        cudaStream_t st);
// C2b for the f1 methods (OFM-f1, TriOFM-f1): only the column dots diag(Z^T Y),
// diag(X^T Y) -> part[nblk][2][KP] (the f1 line search reads T, R' through their
// diagonals alone; kernels_stream.cu k_gram_diag)
int gram_diag_grid(int64_t n);
void launch_gram_diag(ofsc_dtype dt, int KP, int64_t n, const void* Zown, const void* Xown,
                      const void* Y, double* part, const int* stop, int nblk, cudaStream_t st);
// T = diag(diagred[0..KP)), R' = diag(diagred[KP..2KP)) into grams[2..3] (1 CTA)
void launch_expand_diag(const IterParams& p, cudaStream_t st);
// plain SpMM (no Grams) into an arbitrary ld
void launch_spmm_plain(ofsc_dtype dt, int k, int64_t n_local, int64_t own_off,
                       const int64_t* row_ptr, const int32_t* col, const double* s,
                       const float* s32, const void* Zg, int64_t ldz, void* Y, int64_t ldy,
                       cudaStream_t st);
// generic tile Gram pair: part = (A^T B, A^T C) over local rows (KP-padded blocks)
void launch_gram_pair(ofsc_dtype dt, int KP, int64_t n_local, const void* A, const void* B,
                      const void* C, double* part, int nblk, cudaStream_t st);
// sum partial Grams over blocks in fixed order: out[g] = sum_b part[b][g], g < ngram
void launch_reduce_partials(const double* part, int nblk, int per_blk, double* out,
                            cudaStream_t st);
// column partial reduction (gg, dg) -> colred (used when p > 1)
void launch_reduce_cols(const IterParams& p, int nblk, cudaStream_t st);
// beta / convergence / history (1 CTA).  reduced: read colred instead of part_cols
void launch_beta(const IterParams& p, int nblk, int reduced, cudaStream_t st);
// exact line search + algebraic M, W update (1 CTA)
void launch_linesearch(const IterParams& p, cudaStream_t st);
// fixed-order reduction of nblk partial (T, R') arrays into grams[2..3] fused with the
// line search: the last CTA to finish its slice runs it (p == 1).  diag: the partials
// are k_gram_diag's column dots, expanded into diagonal T, R' before the line search
void launch_reduce_linesearch(const IterParams& p, const double* part, int nblk, int diag,
                              cudaStream_t st);
// line-search hook: coefficients from given Grams (device), no ctl
void launch_linesearch_hook(int method, int k, int KP, const double* grams, double* M, double* W,
                            double* alpha, int* codes, cudaStream_t st);
// Rayleigh-Ritz post-step (kernels_rr.cu): k x k solve (1 CTA) and the row pass
void launch_rr_small(const double* M, const double* W, int KP, int k, double* Tm, double* theta,
                     int* status, cudaStream_t st);
int rr_rows_blocks(int64_t n);
void launch_rr_rows(ofsc_dtype dt, int64_t n, int k, int KP, const void* X, const void* AX,
                    const double* Tm, const double* theta, void* U, double* part, int nblk,
                    cudaStream_t st);
// layout helpers
// dst row r <- src row perm[r] (perm may be NULL: identity)
void launch_copy_in(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, int64_t lds,
                    void* dst, const int32_t* perm, cudaStream_t st);
// dst row perm[r] <- src row r (perm may be NULL: identity)
void launch_copy_out(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, void* dst,
                     int64_t ldd, const int32_t* perm, cudaStream_t st);
void launch_row_normalize(ofsc_dtype dt, int64_t n, int k, const void* X, int64_t ldx, void* Y,
                          int64_t ldy, cudaStream_t st);
// K-means
void launch_kmeans_assign(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                          const double* C, int* labels, unsigned long long* changes,
                          double* part_inertia, int nblk, cudaStream_t st);
void launch_kmeans_partial(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                           const int* labels, double* part, int nblk, cudaStream_t st);
void launch_kmeans_finish(int K, int dim, const double* red, double* C, cudaStream_t st);
int kmeans_blocks(int64_t n);
// Fused Lloyd step (assign + per-CTA partial sums, part[nblk][K][dim + 1]); dim <= 64, K <= 128.
bool kmeans_step_supported(int dim, int K);
int kmeans_step_blocks(int64_t n);
// lbound[n]: per-row lower bound on the distance to the nearest other centroid
// (written every step); delta[K]: centroid moves of the last update, NULL on the
// first step (no bounds yet: every row is assigned by the products).
void launch_kmeans_step(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                        const double* C, int* labels, unsigned long long* changes,
                        double* part_inertia, double* part, double* lbound, const double* delta,
                        const double* sep, double* ubound, int nblk, cudaStream_t st);
// light step (bounds first; Y read only by the rows that fail; sums by label changes):
// part[b] = per-CTA (dS, dcnt); ubound/lbound carried from the previous step
bool kmeans_light_supported(int dim, int K);
int kmeans_light_blocks(int64_t n);
void launch_kmeans_light(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                         const double* C, int* labels, double* ubound, double* lbound,
                         const double* delta, const double* sep, unsigned long long* changes,
                         double* part, int nblk, cudaStream_t st);
void launch_kmeans_accum(int n, double* S, const double* dS, cudaStream_t st);
void launch_kmeans_inertia(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy,
                           const double* C, const int* labels, double* part, int nblk,
                           cudaStream_t st);
// sep[c] = half the distance of centroid c to its nearest other centroid (deflated)
void launch_kmeans_halfsep(int K, int dim, const double* C, double* sep, cudaStream_t st);
// fused path: C = means (empty keeps), delta[c] = ||C_new - C_old|| (dim <= 64)
void launch_kmeans_finish_delta(int K, int dim, const double* red, double* C, double* delta,
                                cudaStream_t st);
int kmeans_partial_blocks(int64_t n);

// graph build (graph_build.cu)
struct CsrDevice {
  int64_t n = 0, m_kept = 0, nnz = 0, n_loops = 0, n_dups = 0, n_isolated = 0, max_deg = 0;
  double fro2 = 0.0;
  int64_t* row_ptr = nullptr;  // [n+1]
  int32_t* col = nullptr;      // [nnz] global ids
  double* s = nullptr;         // [n]
};
void build_csr(int64_t n, int64_t m, const int64_t* d_src, const int64_t* d_dst, CsrDevice& out,
               cudaStream_t st);
// append a batch of edges (device arrays, ids of the CSR's numbering) in place:
// the result equals build_csr of the concatenated edge list
void append_csr(CsrDevice& csr, int64_t m, const int64_t* d_src, const int64_t* d_dst,
                cudaStream_t st);
// locality reordering (label propagation): perm[new] = old, inv[old] = new
// (also community id per internal row and community start rows, for L2 cache hints)
void lpa_order(const CsrDevice& csr, int sweeps, int32_t* d_perm, int32_t* d_inv, int64_t* n_comm,
               double* intra_frac, int32_t* d_cid, int64_t** d_cstart, cudaStream_t st);
// original -> internal ids; endpoints outside [0, n) map to -1 (rejected by the build)
void relabel_edges(int64_t m, int64_t n, const int64_t* src, const int64_t* dst,
                   const int32_t* inv, int64_t* s2, int64_t* d2, cudaStream_t st);
void scatter_slots(const double* s, int64_t n, double* s_slot, float* s32_slot,
                   const int64_t* d_begins, int p, int64_t slot_rows, cudaStream_t st);
void rebase_row_ptr(const int64_t* in, int64_t rows, int64_t base, int64_t* out, cudaStream_t st);
// halo layout of one rank (p > 1): own rows then the referenced remote rows
struct HaloLayout {
  int64_t n_local = 0, ext_rows = 0, nnz_local = 0, total_send = 0;
  int64_t* row_ptr = nullptr;        // [n_local + 1], from 0
  int32_t* col = nullptr;            // [nnz_local] ext ids
  int64_t* row_ptr_loc = nullptr;    // the same rows split: columns < n_local (own rows) ...
  int32_t* col_loc = nullptr;
  int64_t* row_ptr_rem = nullptr;    // ... and halo columns (>= n_local), each in CSR order
  int32_t* col_rem = nullptr;
  double* s_ext = nullptr;           // [ext_rows]
  float* s32_ext = nullptr;
  int32_t* d_gid = nullptr;          // [ext_rows] global id of each ext row
  std::vector<int32_t> h_gid;
  std::vector<int64_t> recv_cnt, recv_off;   // per peer: rows, first ext row
  std::vector<int64_t> send_cnt, send_off;   // per peer: rows, offset into d_send_idx
  int32_t* d_send_idx = nullptr;     // [total_send] own row index to send (grouped by peer)
};
void build_halo(const CsrDevice& csr, const int64_t* h_begins, const int64_t* d_begins, int p,
                int rank, HaloLayout& out, cudaStream_t st);

// ---- collectives (comm.cu): NCCL, or an in-process local world on one device ----
struct LocalWorld;
std::shared_ptr<LocalWorld> make_local_world(int nranks);
}  // namespace ofsc

struct ofsc_comm_s {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0, device = 0;
  std::shared_ptr<ofsc::LocalWorld> world;   // in-process world (ofsc_comm_create_local_world)
};

namespace ofsc {
// p > 1 with a transport (NCCL or a local world); a bare local test communicator
// (ofsc_comm_create_local) has none: its reductions stay rank-partial
bool comm_active(const ofsc_comm_s* c);
// buf[0..count) <- sum over ranks in rank order (same bits on every rank); gather: p*count scratch
void comm_sum_f64(ofsc_comm_s* c, double* buf, size_t count, double* gather, cudaStream_t s);
void comm_sum_u64(ofsc_comm_s* c, unsigned long long* buf, size_t count,
                  unsigned long long* gather, cudaStream_t s);
// grouped point-to-point: rows [send_off[q], +send_cnt[q]) of sendbuf go to rank q,
// recv_cnt[q] rows from q land at recvbuf row recv_off[q] (row = row_elems elements)
void comm_exchange(ofsc_comm_s* c, ncclDataType_t type, size_t row_elems, size_t elem_bytes,
                   const void* sendbuf, const std::vector<int64_t>& send_cnt,
                   const std::vector<int64_t>& send_off, void* recvbuf,
                   const std::vector<int64_t>& recv_cnt, const std::vector<int64_t>& recv_off,
                   cudaStream_t s);
}  // namespace ofsc

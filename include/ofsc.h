/*
 * libofsc -- orthogonalization-free spectral clustering on B200 (sm_100a).
 *
 * C ABI of the data-parallel hot path of arXiv 2305.10356
 * ("P:n" = /root/reference/PAPER.md line n).
 *
 *   Alg. 1 l.2   build A = L - 2I from an undirected edge list ....... ofsc_graph_build
 *   Alg. 1 l.3   run OFM-f1 / TriOFM-f1 / OFM-f2 / TriOFM-f2 ......... ofsc_run
 *                       (Algorithm 2)
 *   Alg. 1 l.4   normalise each row of the features ................. ofsc_row_normalize
 *   Alg. 1 l.5   Euclidean K-means (Lloyd) ........................... ofsc_kmeans
 *   P:587               ARI / NMI of two labelings (host) .................. ofsc_scores
 *   Alg. 1 end to end   host buffers in, labels out ........................ ofsc_spectral_cluster
 *   P:589, P:596        orthogonalisation + Rayleigh-Ritz, relerr ........... ofsc_rayleigh_ritz
 *   P:584, P:609        streaming: add an edge part to a built graph ........ ofsc_graph_append
 *   kernel-level hooks  SpMM, SpMM + Grams, line search, exchange plan ...... ofsc_graph_apply,
 *                       ofsc_graph_apply_gram, ofsc_line_search, ofsc_graph_exchange_plan
 *
 * Conventions
 *  - Pointers named d_* are CUDA device pointers, h_* are host pointers.  The
 *    caller allocates and owns every array; the library owns the opaque handles
 *    (graph, comm) and their device workspaces (freed by *_destroy).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device work is stream-ordered.  Calls that fill host outputs (reports,
 *    histories, info, *_out) synchronize `stream` before returning.
 *  - Dense blocks (X, Y, features) are row-major with leading dimension ld >= k
 *    (elements), fp64 (OFSC_F64) or fp32 (OFSC_F32).  fp32 means fp32 storage
 *    of the N x k blocks and fp32 SpMM accumulation, with fp64 Grams, column
 *    dots, k x k state and line search.
 *  - Errors: every call returns an ofsc_status; no exception or exit() crosses
 *    the ABI.  ofsc_last_error() gives a thread-local message for the last
 *    failing call.  OFSC_ERR_ARG: null pointer, k < 1, k > n, k > OFSC_MAX_K,
 *    ld < k, bad enum, rank/size mismatch.  OFSC_ERR_RANGE: edge endpoint
 *    outside [0, n).  OFSC_ERR_CUDA / OFSC_ERR_NCCL: runtime failures.
 *    OFSC_ERR_DIVERGED: a non-finite direction or step (X keeps the last
 *    finite iterate).
 *  - Multi-GPU: one process per GPU.  Rows are partitioned contiguously,
 *    balanced by nnz; a rank's row range is ofsc_graph_info.row_begin/row_end
 *    and every d_X / d_Y / d_labels argument is that rank's local row block.
 *    comm == NULL means a single GPU.  Per iteration each rank exchanges only
 *    the rows its peers reference (halo, grouped ncclSend/ncclRecv, overlapped
 *    with the SpMM's own-column part) and all-reduces the k x k Grams and the
 *    column dots.
 *  - No CPU fallback: every numerical step runs in this library's sm_100a kernels.
 */
#ifndef OFSC_H
#define OFSC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OFSC_MAX_K 64

typedef enum {
  OFSC_OK = 0,
  OFSC_ERR_ARG = 1,
  OFSC_ERR_RANGE = 2,
  OFSC_ERR_NOMEM = 3,
  OFSC_ERR_CUDA = 4,
  OFSC_ERR_NCCL = 5,
  OFSC_ERR_DIVERGED = 6,
  OFSC_ERR_STATE = 7
} ofsc_status;

/* The paper's four methods: direction g and line-search cubic(s). */
typedef enum {
  OFSC_OFM_F1 = 0,    /* grad f1 = 4AX + 4XX^TX            eq:gradientf1 P:188-191 */
  OFSC_TRIOFM_F1 = 1, /* g1 = AX + X triu(X^TX)            eq:gradientg1 P:209-212 */
  OFSC_OFM_F2 = 2,    /* grad f2 = 4AX - 2XX^TAX - 2AXX^TX eq:gradientf2 P:232-235 */
  OFSC_TRIOFM_F2 = 3  /* g2 = 2AX - AXtriu(X^TX) - Xtriu(X^TAX) eq:gradientg2 P:250-253 */
} ofsc_method;

typedef enum { OFSC_F64 = 0, OFSC_F32 = 1 } ofsc_dtype;

/* Column-wise CG (Alg. 2 l.9): Polak-Ribiere, PR+ = max(beta, 0), or
 * beta = 0 (steepest descent with exact line search). */
typedef enum { OFSC_BETA_PR = 0, OFSC_BETA_PR_PLUS = 1, OFSC_BETA_ZERO = 2 } ofsc_beta_rule;

typedef struct ofsc_comm_s* ofsc_comm;
typedef struct ofsc_graph_s* ofsc_graph;
typedef void* ofsc_stream;

const char* ofsc_version(void);
const char* ofsc_status_string(ofsc_status s);
const char* ofsc_last_error(void);

/* Device memory held for reuse: the library keeps the buffers of destroyed
 * graphs and finished calls (exact-size block cache, <= OFSC_BLOCK_CACHE_GB,
 * default 40, over the device's stream-ordered pool) so repeated calls with
 * the same shapes allocate nothing.  ofsc_trim_memory synchronises the current
 * device, releases every cached block and trims the pool, returning the memory
 * to other allocators (e.g. PyTorch's).  Not part of any paper step. */
ofsc_status ofsc_trim_memory(void);

/* ---- communicator (NCCL over NVLink/NVSwitch) ---------------------------
 * Rank 0 calls ofsc_get_unique_id and broadcasts the 128 bytes (e.g. with
 * torch.distributed); every rank then calls ofsc_comm_create on its own GPU. */
ofsc_status ofsc_get_unique_id(void* h_id128);
ofsc_status ofsc_comm_create(const void* h_id128, int nranks, int rank, int cuda_device,
                             ofsc_comm* out);
ofsc_status ofsc_comm_destroy(ofsc_comm comm);
/* Test communicator for rank `rank` of `nranks` WITHOUT NCCL: graph build and the
 * kernel hooks (ofsc_graph_apply / _apply_gram) run on this rank's row block with
 * rank-partial reductions; ofsc_run / ofsc_kmeans reject it (OFSC_ERR_STATE).
 * Lets one process check the multi-rank partition and layout on one GPU. */
ofsc_status ofsc_comm_create_local(int nranks, int rank, ofsc_comm* out);
/* In-process world of `nranks` ranks on the CURRENT device, WITHOUT NCCL:
 * h_out[r] (host array of nranks handles, filled) is the communicator of rank
 * r.  Every call of the library then runs the full p > 1 schedule of the
 * row-partitioned multi-GPU path: halo exchange
 * of V / X rows, sums over ranks (all-gather + fixed rank-order sum, the same
 * kernel the NCCL path runs), split SpMM, K-means reductions.  The transport
 * is host barriers + device-to-device copies between the ranks' buffers, so
 * EACH RANK MUST BE DRIVEN BY ITS OWN HOST THREAD (a collective returns only
 * when every rank has reached it) and every rank must make the same sequence
 * of calls.  No kernel waits on another rank's kernel.  Iterations run as
 * eager launches (host barriers cannot be captured in a CUDA graph).  For
 * tests and emulation of the multi-GPU schedule on one GPU; destroy each
 * handle with ofsc_comm_destroy.  OFSC_ERR_ARG: nranks < 1 or h_out NULL. */
ofsc_status ofsc_comm_create_local_world(int nranks, ofsc_comm* h_out);
/* Host-only: contiguous split of rows [0, n) over p ranks with ~equal nnz(A)
 * = sum_i (deg_i + 1), from CSR offsets h_row_ptr[n+1]; h_begins[p+1] out. */
ofsc_status ofsc_partition_rows(int64_t n, const int64_t* h_row_ptr, int p, int64_t* h_begins);

/* ---- graph -> operator A = L - 2I (Alg. 1 l.2) ----------
 * Canonical undirected edge set: self-loops dropped, duplicates collapsed
 * (S_ij in {0,1}); d_i = |N(i)|, s_i = d_i^{-1/2} (0 if isolated);
 * A_ii = -1, A_ij = -s_i s_j.  The CSR pattern (int64 row offsets, int32
 * column ids sorted ascending per row) and s live on the device; values of A
 * are implicit.  src/dst: m edges, host (edges_on_device = 0) or device
 * pointers; every rank passes the full edge list.  Requires 1 <= n < 2^31. */
typedef struct {
  int64_t n;                    /* nodes */
  int64_t n_edges_kept;         /* unique undirected non-loop edges */
  int64_t nnz_global;           /* 2 * n_edges_kept (off-diagonal nnz of S) */
  int64_t row_begin, row_end;   /* this rank's rows [row_begin, row_end) */
  int64_t nnz_local;            /* off-diagonal nnz in this rank's rows */
  int64_t n_isolated;           /* nodes with d_i = 0 */
  int64_t n_self_loops_dropped;
  int64_t n_duplicates_dropped;
  int64_t max_degree;
  double fro2_A;                /* ||A||_F^2 = n + sum_ij (s_i s_j)^2 */
  double load_imbalance;        /* p * max_r nnz_r / nnz */
  int32_t reordered;            /* 1 if rows were reordered by ofsc_build_opts.reorder */
  int64_t n_communities;        /* label-propagation communities (reordered graphs) */
  double intra_edge_fraction;   /* fraction of nnz joining two nodes of one community */
  int64_t halo_rows;            /* p > 1: remote rows this rank's columns reference */
  int64_t send_rows;            /* p > 1: own rows sent to peers per exchange (sum over peers) */
} ofsc_graph_info;

/* Build options.  reorder = 1: a locality reordering of the rows derived from
 * the graph itself (semi-synchronous label propagation, `lpa_sweeps` sweeps;
 * nodes ordered by (community, id)) so the SpMM's neighbour gathers hit L2.
 * The operator is the same matrix with permuted rows/columns (P A P^T); the
 * mathematics of every call is unchanged.  Internal row i is node perm[i]
 * (ofsc_graph_copy_perm).  With p == 1, ofsc_run / ofsc_graph_apply(_gram)
 * take and return rows in the caller's ORIGINAL node order (the library
 * permutes); with p > 1, a rank's local rows are internal rows
 * [row_begin, row_end), i.e. nodes perm[row_begin .. row_end). */
typedef struct {
  int32_t reorder;     /* 0 = keep node ids (default of ofsc_graph_build), 1 = LPA reorder */
  int32_t lpa_sweeps;  /* max sweeps (<= 0: 30); stops early when < n/1000 labels change */
} ofsc_build_opts;

ofsc_status ofsc_graph_build(ofsc_comm comm, int64_t n, int64_t m, const int64_t* src,
                             const int64_t* dst, int edges_on_device, ofsc_stream stream,
                             ofsc_graph* out);
ofsc_status ofsc_graph_build_ex(ofsc_comm comm, int64_t n, int64_t m, const int64_t* src,
                                const int64_t* dst, int edges_on_device,
                                const ofsc_build_opts* bopts, ofsc_stream stream, ofsc_graph* out);
ofsc_status ofsc_graph_info_get(ofsc_graph g, ofsc_graph_info* out);
/* Copy this rank's CSR to host: h_row_ptr[n_local+1] (offsets from 0),
 * h_col[nnz_local] (internal global ids), h_s[n] (internal order). Any pointer may be NULL. */
ofsc_status ofsc_graph_copy_csr(ofsc_graph g, int64_t* h_row_ptr, int32_t* h_col, double* h_s);
/* h_perm[n]: internal row -> original node id (identity unless reordered). */
ofsc_status ofsc_graph_copy_perm(ofsc_graph g, int32_t* h_perm);
ofsc_status ofsc_graph_destroy(ofsc_graph g);

/* Multi-GPU exchange plan of this rank (p > 1):
 * the gather buffer holds the rank's own rows then its halo -- the remote rows
 * its columns reference, ascending global id.  Per exchange the rank sends to
 * peer q the own rows that have a neighbour in q's range (h_send_gids, grouped
 * by q, ascending) and receives from q its halo segment (h_recv_gids).  Both
 * sides derive the plan from the symmetric graph, so q's send list to r equals
 * r's receive list from q.  Counts are per peer [p]; id arrays hold
 * info.send_rows / info.halo_rows global ids (internal row order).  Any output
 * may be NULL.  p == 1: all counts are 0. */
ofsc_status ofsc_graph_exchange_plan(ofsc_graph g, int64_t* h_send_counts, int32_t* h_send_gids,
                                     int64_t* h_recv_counts, int32_t* h_recv_gids);

/* Streaming: append a batch of undirected edges to
 * a built graph in place, so that it equals the graph built from the
 * concatenation of all batches (same CSR, s = D^{-1/2}, ||A||_F^2 and counts,
 * bit for bit).  New edges are sorted and deduplicated on the device and merged
 * row by row into the existing CSR (no re-sort of the old edges).  Endpoints use
 * the original node ids; a reordered graph keeps its row order (the new edges
 * are relabelled into it).  Node count n is fixed (snapshots of a graph with
 * known n, as in the Graph Challenge streams).  Invalidates the run workspace.
 * Single-rank graphs only (OFSC_ERR_STATE when p > 1: rebuild instead).
 * OFSC_ERR_RANGE for an endpoint outside [0, n), graph unchanged. */
ofsc_status ofsc_graph_append(ofsc_graph g, int64_t m, const int64_t* src, const int64_t* dst,
                              int edges_on_device, ofsc_stream stream);

/* Y = A Z for this rank's rows (the SpMM of eq:spmm P:440, values implicit).
 * d_Z: all n rows (n x ldz, original node order) on every rank; d_Y: local
 * rows (n_local x ldy; original order when p == 1, internal order when p > 1). */
ofsc_status ofsc_graph_apply(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_Z,
                             int64_t ldz, void* d_Y, int64_t ldy, ofsc_stream stream);

/* Kernel-level hook of the SpMM + Gram step (the SpMM kernel C2a, then the
 * TMA-streamed DMMA Gram kernel C2b): Y = A Z (local rows) and
 * the k x k fp64 Grams d_grams[0..3] = Z^T Z, Z^T X, Z^T Y, X^T Y (row-major,
 * 4 consecutive k x k blocks, summed over all ranks).  Z: n x ldz (all rows),
 * X: local rows x ldx. */
ofsc_status ofsc_graph_apply_gram(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_Z,
                                  int64_t ldz, const void* d_X, int64_t ldx, void* d_Y,
                                  int64_t ldy, double* d_grams, ofsc_stream stream);

/* ---- the orthogonalization-free iteration (Algorithm 2) ----- */
typedef struct {
  int32_t k;            /* features, 1 <= k <= min(n, OFSC_MAX_K) */
  int32_t max_iters;    /* T: number of updates of X (tol = 0 runs exactly T) */
  double tol;           /* 0 => fixed T (paper protocol); else stop when
                           ||G||_F <= tol * c_m * ||X||_F, c_m = 4,1,2,1 */
  int32_t beta_rule;    /* ofsc_beta_rule, default OFSC_BETA_PR_PLUS */
  int32_t line_search;  /* 1 = exact line search; 0 = alpha_fixed */
  double alpha_fixed;
  int32_t refresh;      /* 1 = paper schedule: AX, X^TX, X^TAX recomputed every
                           iteration (2 SpMMs); R > 1: recurrence
                           AX += AV diag(alpha) + algebraic k x k update, recompute
                           every R iterations; 0 = never recompute */
  int32_t check_every;  /* with tol > 0: poll the device stop flag every n iterations */
  int32_t timing_skip;  /* >= 0: CUDA-event time iterations [timing_skip, iters) on `stream`
                           into ofsc_report.timed_ms; < 0: off */
  int32_t profile;      /* 1: per-kernel CUDA-event timing into ofsc_report.kernel_ms
                           (launches not captured in a CUDA graph); 0: off */
} ofsc_opts;

void ofsc_opts_default(ofsc_opts* o); /* k=0 (must be set), T=100, tol=0, PR+, exact LS,
                                         refresh=0, check_every=8, timing_skip=-1, profile=0 */

/* Kernel phases of one iteration, indices of ofsc_report.kernel_ms / kernel_launches. */
enum {
  OFSC_PH_UPDATE_DIRECTION = 0, /* C3: X += aV, AX += aAV, G = g_m(X), column dots */
  OFSC_PH_BETA = 1,             /* k x k: beta, ||G||, objective, stop flags */
  OFSC_PH_DIRECTION_GRAM = 2,   /* C4: V = -G + beta Vp, Q = V^T V, P = V^T X */
  OFSC_PH_SPMM_GRAM = 3,        /* C2a: AV = A V (neighbour gathers) */
  OFSC_PH_GRAM_REDUCE = 4,      /* fixed-order reduction of per-CTA Gram partials */
  OFSC_PH_LINE_SEARCH = 5,      /* k x k: cubics, roots, alpha, M/W update */
  OFSC_PH_REFRESH = 6,          /* refresh iterations: X update, A X, X^T X, X^T A X */
  OFSC_PH_COMM = 7,             /* NCCL collectives (p > 1) */
  OFSC_PH_GRAM_STREAM = 8,      /* C2b: T = V^T AV, R' = X^T AV (TMA-streamed, DMMA);
                                   OFM-f1 / TriOFM-f1: diag T, diag R' only (their cubics,
                                   P:298-305 and P:315-322, read no other entry) */
  OFSC_NUM_PHASES = 10
};

typedef struct {
  int32_t iters;              /* completed updates of X */
  int32_t converged;          /* 1 if ||G|| hit the tolerance (or 0) */
  int32_t diverged;           /* 1 if a direction or step was non-finite */
  int32_t n_three_root_steps; /* line searches that selected among 3 real roots */
  int32_t n_zero_steps;       /* degenerate (all-zero) cubics, alpha = 0 */
  double grad_norm0, grad_norm, objective;
  int32_t timed_iters;        /* iterations inside the timing window */
  int32_t launches;           /* kernels this library launched inside the timing window */
  double timed_ms;            /* CUDA-event time of the timing window (opts.timing_skip) */
  double kernel_ms[10];        /* opts.profile: summed per-phase kernel time in the window */
  int32_t kernel_launches[10]; /* opts.profile: launches per phase in the window */
} ofsc_report;

/* d_X (local rows x ldx, dtype dt): in = X0 or a warm start, out = features.
 * h_history (optional, max_iters x 4): per iteration objective f(X_t), ||G_t||_F,
 * min alpha_t, max alpha_t (NaN after a stop).  Synchronizes `stream`. */
ofsc_status ofsc_run(ofsc_graph g, ofsc_method method, ofsc_dtype dt, const ofsc_opts* opts,
                     void* d_X, int64_t ldx, double* h_history, ofsc_report* rep,
                     ofsc_stream stream);
/* As ofsc_run, plus optional per-iteration step sizes and root-branch codes
 * (host, max_iters x k each; codes as in DESIGN.md R9). */
ofsc_status ofsc_run_ex(ofsc_graph g, ofsc_method method, ofsc_dtype dt, const ofsc_opts* opts,
                        void* d_X, int64_t ldx, double* h_history, double* h_alphas,
                        int32_t* h_codes, ofsc_report* rep, ofsc_stream stream);

/* Kernel-level hook of the k x k exact line search (1 CTA on the device):
 * given host Grams Q, P, T, R' = X^TAV, M = X^TX, W = X^TAX (k x k row-major
 * each), return per-column alpha and branch codes (OFM methods broadcast
 * one alpha) and the algebraically updated M, W (may be NULL). */
ofsc_status ofsc_line_search(ofsc_method method, int32_t k, const double* h_Q, const double* h_P,
                             const double* h_T, const double* h_Rp, const double* h_M,
                             const double* h_W, double* h_alpha, int32_t* h_codes,
                             double* h_M_out, double* h_W_out);

/* ---- post-processing (Alg. 1 l.4-5) ------------------------------------- */
/* y_i = x_i / ||x_i||_2, a zero row stays zero.  In-place allowed. */
ofsc_status ofsc_row_normalize(ofsc_dtype dt, int64_t n_local, int32_t k, const void* d_X,
                               int64_t ldx, void* d_Y, int64_t ldy, ofsc_stream stream);

/* Lloyd K-means from given centroids d_centroids (K x dim fp64, in: init,
 * out: final).  Assign: argmin_c sum_{d<dim} (y_d - C_cd)^2 (fp64, summed in
 * d order, ties -> lowest c); update: cluster means (empty cluster keeps its
 * centroid); stop when no label changes or after max_iters assignments.
 * d_labels: int32 local rows; 1 <= n_clusters <= 128.  iters_out / inertia_out optional host outputs. */
ofsc_status ofsc_kmeans(ofsc_comm comm, ofsc_dtype dt, int64_t n_local, int32_t dim,
                        const void* d_Y, int64_t ldy, int32_t n_clusters, double* d_centroids,
                        int32_t max_iters, int32_t* d_labels, int32_t* iters_out,
                        double* inertia_out, ofsc_stream stream);

/* Orthogonalisation + Rayleigh-Ritz post-step and the relerr metric
 * ("one SpMM, several dot products, and an eigendecomposition of a
 * k x k matrix"; relerr = ||B U - U Lambda||_F / ||U Lambda||_F with
 * B = L + 2I = A + 4I, R24-R26).
 *   A X (one SpMM), M = X^T X, W = X^T A X; M = L L^T (Cholesky-QR, Q = X L^{-T});
 *   H = L^{-1} ((W + W^T)/2) L^{-T} = Z Theta Z^T (k x k Jacobi on device);
 *   U = X L^{-T} Z (Ritz vectors, orthonormal), A U = (A X) L^{-T} Z.
 * d_X: local rows x ldx (original node order when p == 1), dtype dt, not modified.
 * d_U: optional (NULL: not written) local rows x ldu, same order and dtype.
 * h_theta: host [k], Ritz values of A ascending (those of B are theta + 4).
 * h_relerr: optional host scalar.  Synchronizes the stream.
 * Errors: OFSC_ERR_ARG (k < 1, k > min(n, OFSC_MAX_K), ld < k, null X/theta);
 * OFSC_ERR_RANGE when X^T X is not positive definite (X rank deficient). */
ofsc_status ofsc_rayleigh_ritz(ofsc_graph g, ofsc_dtype dt, int32_t k, const void* d_X,
                               int64_t ldx, void* d_U, int64_t ldu, double* h_theta,
                               double* h_relerr, ofsc_stream stream);

/* ARI and NMI (arithmetic-mean normalisation) of two host labelings. */
ofsc_status ofsc_scores(int64_t n, const int32_t* h_a, const int32_t* h_b, double* ari,
                        double* nmi);

/* Algorithm 1 end to end from HOST buffers: edges (m, full list) -> build A
 * (bopts NULL: LPA locality reordering iff opts->max_iters >= 32) -> run `method` from h_X
 * (ALL n rows x k in original node order, dense ld = k, dtype dt; in: X0, out:
 * features before normalisation for the nodes this rank owns) -> row-normalise
 * -> K-means with centroids initialised at the original node ids
 * h_init_rows[n_clusters] of the normalised features -> h_labels[n] (filled
 * for the nodes this rank owns).  Copies host<->device inside the call. */
ofsc_status ofsc_spectral_cluster(ofsc_comm comm, int64_t n, int64_t m, const int64_t* h_src,
                                  const int64_t* h_dst, ofsc_method method, ofsc_dtype dt,
                                  const ofsc_opts* opts, const ofsc_build_opts* bopts, void* h_X,
                                  int32_t n_clusters, const int64_t* h_init_rows,
                                  int32_t km_max_iters, int32_t* h_labels, ofsc_report* rep,
                                  ofsc_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* OFSC_H */

// Lloyd K-means on the normalised features (Alg. 1 l.5).
//   assign: label_r = argmin_c sum_{d=0}^{dim-1} (y_rd - C_cd)^2, summed in d
//           order in fp64, ties -> lowest c (R20).  Compiled with
//           -fmad=false so the distance rounds exactly as written, identical to
//           the oracle's, and every argmin decision is taken in the same precision.
//   update: per-CTA partial sums over a contiguous row range in row order (one
//           thread per feature column, no atomics), fixed-order reduction,
//           mean; an empty cluster keeps its centroid.
#include <math_constants.h>

#include "common.cuh"
#include "sm100.cuh"

namespace ofsc {

constexpr int kKmThreads = 256;

// One warp per group of KR rows; lane l evaluates centroids l, l+32, ... (KC per
// lane) for all KR rows at once (KR*KC independent accumulation chains, each
// summed in d order); centroids are held transposed in smem (Ct[d][c]) so a
// warp's reads are conflict-free and each Ct element is reused KR times.
constexpr int kKmRows = 4;

template <typename T, int KC>
__global__ void __launch_bounds__(kKmThreads)
k_kmeans_assign(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy, int K,
                const double* __restrict__ C, int* __restrict__ labels,
                unsigned long long* changes, double* part_inertia) {
  constexpr int KR = kKmRows;
  extern __shared__ double sm[];
  double* Ct = sm;                         // [dim][K]
  double* rows = Ct + (size_t)dim * K;     // [8 warps][KR][dim]
  __shared__ double s_in[kKmThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < dim * K; e += kKmThreads) {
    const int c = e / dim, d = e % dim;
    Ct[d * K + c] = C[e];
  }
  __syncthreads();
  double* yr = rows + (size_t)warp * KR * dim;
  double inertia = 0.0;
  unsigned long long nchg = 0;
  const int64_t nw = (int64_t)gridDim.x * (kKmThreads / 32);
  for (int64_t r0 = ((int64_t)blockIdx.x * (kKmThreads / 32) + warp) * KR; r0 < n; r0 += nw * KR) {
    for (int e = lane; e < KR * dim; e += 32) {
      const int q = e / dim, d = e % dim;
      yr[e] = r0 + q < n ? ld1(Y + (r0 + q) * ldy + d) : 0.0;
    }
    __syncwarp();
    double acc[KR][KC];
#pragma unroll
    for (int q = 0; q < KR; ++q)
#pragma unroll
      for (int j = 0; j < KC; ++j) acc[q][j] = 0.0;
    for (int d = 0; d < dim; ++d) {
      double cv[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        const int c = lane + 32 * j;
        cv[j] = c < K ? Ct[d * K + c] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        const double y = yr[q * dim + d];
#pragma unroll
        for (int j = 0; j < KC; ++j) {
          const double diff = y - cv[j];
          acc[q][j] = acc[q][j] + diff * diff;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < KR; ++q) {
      double best = 0.0;
      int bc = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        const int c = lane + 32 * j;
        if (c < K && (bc == 0x7fffffff || acc[q][j] < best)) {  // c increases: lowest index wins ties
          best = acc[q][j];
          bc = c;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (oc != 0x7fffffff && (bc == 0x7fffffff || ob < best || (ob == best && oc < bc))) {
          best = ob;
          bc = oc;
        }
      }
      const int64_t r = r0 + q;
      if (lane == 0 && r < n) {
        if (labels[r] != bc) ++nchg;
        labels[r] = bc;
        inertia += best;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    s_in[warp] = inertia;
    if (nchg) atomicAdd(changes, nchg);      // integer: order-independent
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < kKmThreads / 32; ++w) a += s_in[w];
    part_inertia[blockIdx.x] = a;
  }
}

int kmeans_partial_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

int kmeans_blocks(int64_t n) {
  int64_t b = (n + 63) / 64;
  const int64_t cap = (int64_t)num_sms() * 4;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename T, int KC>
static void launch_assign_kc(int64_t n, int dim, const T* Y, int64_t ldy, int K, const double* C,
                             int* labels, unsigned long long* changes, double* part_inertia,
                             int nblk, size_t smem, cudaStream_t st) {
  OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_assign<T, KC>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_kmeans_assign<T, KC><<<nblk, kKmThreads, smem, st>>>(n, dim, Y, ldy, K, C, labels, changes,
                                                         part_inertia);
  OFSC_LAUNCH_CHECK();
}

template <typename T>
static void launch_assign_t(int64_t n, int dim, const T* Y, int64_t ldy, int K, const double* C,
                            int* labels, unsigned long long* changes, double* part_inertia,
                            int nblk, size_t smem, cudaStream_t st) {
  const int kc = (K + 31) / 32;
  if (kc <= 1) launch_assign_kc<T, 1>(n, dim, Y, ldy, K, C, labels, changes, part_inertia, nblk, smem, st);
  else if (kc == 2) launch_assign_kc<T, 2>(n, dim, Y, ldy, K, C, labels, changes, part_inertia, nblk, smem, st);
  else if (kc == 3) launch_assign_kc<T, 3>(n, dim, Y, ldy, K, C, labels, changes, part_inertia, nblk, smem, st);
  else if (kc == 4) launch_assign_kc<T, 4>(n, dim, Y, ldy, K, C, labels, changes, part_inertia, nblk, smem, st);
  else throw Error{OFSC_ERR_ARG, "n_clusters > 128 not supported"};
}

// ---------------------------------------------------------------------------
// Tensor-core assignment with an exactness guard.  Scores s_c = ||c||^2 - 2 y.c
// come from DMMA (y.c for 8 rows x 8 centroids per mma, fp64); argmin_c s_c is
// argmin_c ||y - c||^2.  The oracle's decision is taken on the direct form
// sum_d (y_d - c_d)^2 summed in d order; both forms are within
// tau = 1e-12 (1 + ||y||^2) of the exact distances for unit-norm-scale data
// (dim <= 64: (dim + 2) u ||y - c||^2 and 2 dim u (||y||^2 + ||c||^2)), so when
// the best score beats the runner-up by more than tau the label equals the
// oracle's; otherwise the row falls back to the direct form over all centroids
// (same arithmetic as the oracle, ties -> lowest index).  Labels are therefore
// the oracle's; only the inertia of guarded rows uses the score form.
// ---------------------------------------------------------------------------
template <typename T, int KB>
__global__ void __launch_bounds__(kKmThreads)
k_kmeans_assign_mma(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy, int K,
                    const double* __restrict__ C, int* __restrict__ labels,
                    unsigned long long* changes, double* part_inertia) {
  constexpr int KP = KB * 8;
  constexpr int LDC = KP + 4;
  extern __shared__ double sm[];
  const int DP = (dim + 3) & ~3;
  const int LDY = DP + 4;
  double* Ct = sm;                               // [DP][LDC]  B[k=d][n=c] = C[c][d]
  double* cn = Ct + (size_t)DP * LDC;            // [KP] ||c||^2 (inf for padding)
  double* Ys = cn + KP;                          // [8 warps][8][LDY]
  __shared__ double s_in[kKmThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  for (int e = tid; e < DP * LDC; e += kKmThreads) {
    const int d = e / LDC, c = e % LDC;
    Ct[e] = (c < K && d < dim) ? C[c * dim + d] : 0.0;
  }
  for (int c = tid; c < KP; c += kKmThreads) {
    double a = 0.0;
    if (c < K)
      for (int d = 0; d < dim; ++d) a = a + C[c * dim + d] * C[c * dim + d];
    cn[c] = c < K ? a : CUDART_INF;
  }
  __syncthreads();
  double* ys = Ys + (size_t)warp * 8 * LDY;
  double inertia = 0.0;
  unsigned long long nchg = 0;
  const int64_t nw = (int64_t)gridDim.x * (kKmThreads / 32);
  // the next 8-row group is loaded into registers while the current one computes
  double pre[16];
  auto fetch = [&](int64_t rr) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int e = lane + 32 * j;
      if (e < 8 * DP) {
        const int q = e / DP, d = e % DP;
        pre[j] = (rr + q < n && d < dim) ? ld1(Y + (rr + q) * ldy + d) : 0.0;
      }
    }
  };
  int64_t r0 = ((int64_t)blockIdx.x * (kKmThreads / 32) + warp) * 8;
  if (r0 < n) fetch(r0);
  for (; r0 < n; r0 += nw * 8) {
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int e = lane + 32 * j;
      if (e < 8 * DP) ys[(e / DP) * LDY + (e % DP)] = pre[j];
    }
    __syncwarp();
    if (r0 + nw * 8 < n) fetch(r0 + nw * 8);
    double acc[KB][2];
#pragma unroll
    for (int b = 0; b < KB; ++b) acc[b][0] = acc[b][1] = 0.0;
    for (int d0 = 0; d0 < DP; d0 += 4) {
      const double a = ys[gid * LDY + d0 + tig];
      const double* brow = Ct + (d0 + tig) * LDC + gid;
#pragma unroll
      for (int b = 0; b < KB; ++b) dmma(acc[b][0], acc[b][1], a, brow[b * 8]);
    }
    // lane: row gid, centroids b*8 + 2 tig + h
    double b1 = CUDART_INF, b2 = CUDART_INF;
    int c1 = 0x7fffffff;
#pragma unroll
    for (int b = 0; b < KB; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = b * 8 + 2 * tig + h;
        const double sc = cn[c] - 2.0 * acc[b][h];
        if (sc < b1 || (sc == b1 && c < c1)) {
          b2 = b1;
          b1 = sc;
          c1 = c;
        } else if (sc < b2) {
          b2 = sc;
        }
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {                 // merge the 4 lanes of the row
      const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
      const double ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
      const int oc1 = __shfl_xor_sync(0xffffffffu, c1, o);
      if (ob1 < b1 || (ob1 == b1 && oc1 < c1)) {
        b2 = fmin(b1, ob2);
        b1 = ob1;
        c1 = oc1;
      } else {
        b2 = fmin(b2, ob1);
      }
    }
    double yn = 0.0;                                   // ||y||^2 of row gid
    for (int d = tig; d < DP; d += 4) yn = yn + ys[gid * LDY + d] * ys[gid * LDY + d];
    yn += __shfl_xor_sync(0xffffffffu, yn, 1);
    yn += __shfl_xor_sync(0xffffffffu, yn, 2);
    const int64_t r = r0 + gid;
    const bool guard = !(b2 - b1 > 1e-12 * (1.0 + yn));
    int lab = c1;
    double dist = yn + b1;
    if (guard) {                                       // direct form, exactly as the oracle
      double best = CUDART_INF;
      int bc = 0x7fffffff;
      for (int c = tig; c < K; c += 4) {
        double a = 0.0;
        for (int d = 0; d < dim; ++d) {
          const double diff = ys[gid * LDY + d] - C[c * dim + d];
          a = a + diff * diff;
        }
        if (a < best || (a == best && c < bc)) {
          best = a;
          bc = c;
        }
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ob < best || (ob == best && oc < bc)) {
          best = ob;
          bc = oc;
        }
      }
      lab = bc;
      dist = best;
    }
    if (tig == 0 && r < n) {
      if (labels[r] != lab) ++nchg;
      labels[r] = lab;
      inertia += dist;
    }
    __syncwarp();
  }
  // warp sums: lanes with tig == 0 hold row partials
  for (int o = 16; o; o >>= 1) {
    inertia += __shfl_xor_sync(0xffffffffu, inertia, o);
    nchg += __shfl_xor_sync(0xffffffffu, nchg, o);
  }
  if (lane == 0) {
    s_in[warp] = inertia;
    if (nchg) atomicAdd(changes, nchg);
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < kKmThreads / 32; ++w) a += s_in[w];
    part_inertia[blockIdx.x] = a;
  }
}

template <typename T, int KB>
static void launch_mma_kb(int64_t n, int dim, const T* Y, int64_t ldy, int K, const double* C,
                          int* labels, unsigned long long* changes, double* part_inertia, int nblk,
                          cudaStream_t st) {
  const int DP = (dim + 3) & ~3;
  const size_t smem = ((size_t)DP * (KB * 8 + 4) + KB * 8 + (size_t)8 * 8 * (DP + 4)) * 8;
  OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_assign_mma<T, KB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_kmeans_assign_mma<T, KB><<<nblk, kKmThreads, smem, st>>>(n, dim, Y, ldy, K, C, labels, changes,
                                                              part_inertia);
  OFSC_LAUNCH_CHECK();
}

template <typename T>
static bool launch_mma_t(int64_t n, int dim, const T* Y, int64_t ldy, int K, const double* C,
                         int* labels, unsigned long long* changes, double* part_inertia, int nblk,
                         cudaStream_t st) {
  if (dim > 64) return false;
  const int kb = (K + 7) / 8;
#define OFSC_KB(NB)                                                                             \
  case NB:                                                                                      \
    launch_mma_kb<T, NB>(n, dim, Y, ldy, K, C, labels, changes, part_inertia, nblk, st);        \
    return true;
  switch (kb) {
    OFSC_KB(1) OFSC_KB(2) OFSC_KB(3) OFSC_KB(4) OFSC_KB(5) OFSC_KB(6) OFSC_KB(7) OFSC_KB(8)
    OFSC_KB(9) OFSC_KB(10) OFSC_KB(11) OFSC_KB(12) OFSC_KB(13) OFSC_KB(14) OFSC_KB(15) OFSC_KB(16)
    default: return false;
  }
#undef OFSC_KB
}

void launch_kmeans_assign(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                          const double* C, int* labels, unsigned long long* changes,
                          double* part_inertia, int nblk, cudaStream_t st) {
  const size_t smem =
      ((size_t)dim * K + (size_t)(kKmThreads / 32) * kKmRows * dim) * sizeof(double);
  OFSC_REQUIRE(smem <= 200 * 1024, OFSC_ERR_ARG, "n_clusters * dim too large for K-means smem");
  static int use_mma = -1;
  if (use_mma < 0) {
    const char* e = getenv("OFSC_KMEANS_DIRECT");   // 1: plain direct-form kernel only
    use_mma = (e && e[0] == '1') ? 0 : 1;
  }
  if (use_mma) {
    if (dt == OFSC_F64 && launch_mma_t<double>(n, dim, (const double*)Y, ldy, K, C, labels, changes,
                                                part_inertia, nblk, st))
      return;
    if (dt == OFSC_F32 && launch_mma_t<float>(n, dim, (const float*)Y, ldy, K, C, labels, changes,
                                               part_inertia, nblk, st))
      return;
  }
  if (dt == OFSC_F64)
    launch_assign_t<double>(n, dim, (const double*)Y, ldy, K, C, labels, changes, part_inertia,
                            nblk, smem, st);
  else
    launch_assign_t<float>(n, dim, (const float*)Y, ldy, K, C, labels, changes, part_inertia,
                           nblk, smem, st);
}

// ---------------------------------------------------------------------------
// Fused Lloyd step (dim <= 64, K <= 128): assignment + per-CTA partial sums in
// one pass over Y.  A CTA walks 32-row tiles (static stride, so the summation
// order is fixed); the tile is staged in padded smem (next tile prefetched into
// registers).
//   skip test (steps >= 2; Hamerly's bounds, exact decisions): every row keeps a
//           lower bound lb_r <= min_{c != a} ||y_r - c|| for its label a.  After
//           the centroids moved by delta_c (triangle inequality) it becomes
//           lb_r - max_{c != a} delta_c; the distance to the own centroid is
//           recomputed directly (d order, 8 lanes).  If sqrt(D_a) (1 + rel) <
//           lb (rel = 1e-12 >> the (dim + 2) u rounding of either side's
//           distances), every other centroid is strictly farther in the
//           oracle's arithmetic too, so its argmin is a: the row keeps its
//           label and its distance, and needs no assignment products.
//   assign: only for 8-row blocks holding a row that failed the test.  Warp w
//           owns centroid blocks w (and w + 8); its DMMA B fragments (C^T, DP/4
//           k-steps) stay in registers; scores ||c||^2 - 2 y.c; best /
//           runner-up merged across lanes and warps (8 threads per row,
//           butterfly; the merge is the lexicographic (score, index) minimum,
//           so ties go to the lowest index); the same exactness guard as
//           k_kmeans_assign_mma (direct form in d order when the margin is
//           below tau).  The runner-up score gives the row's new lower bound.
//   sums:   S[c][d] += Y[r][d] for label_r = c, by the warp owning c (lane l:
//           columns 2l, 2l + 1), rows in tile order: fixed order, no atomics,
//           deterministic.  Counts: integer smem atomics (exact).
// part[b] = (sums, count) per centroid feeds the fixed-order reduction.
// ---------------------------------------------------------------------------
constexpr int kKsRows = 32;
constexpr int kKsStages = 3;
static_assert(kKsRows == 32, "the row-mask logic maps tile rows to lanes");
constexpr double kKmRel = 1e-12;   // relative margin of the bound tests

// Scores of NBLK compacted 8-row blocks against this warp's centroid blocks:
// best / runner-up (score, index) per row slot, merged over the row's 4 lanes.
template <int NBLK, int NBW, int DP>
__device__ __forceinline__ void km_assign_blocks(const double* Ys, const int (&rowA)[4],
                                                 const double (&bf)[NBW][DP / 4],
                                                 const double* cn, int warp, int KB, int tig,
                                                 double (&b1)[4], double (&b2)[4], int (&c1)[4]) {
  constexpr int LDY = DP + 4;
  // CH independent accumulation chains per block (k-steps kk = ch mod CH), so a
  // single block is not one 16-deep dependent DMMA chain
  constexpr int CH = NBLK >= 4 ? 1 : (NBLK == 3 ? 1 : 4 / NBLK);
#pragma unroll
  for (int q = 0; q < NBW; ++q) {
    const int cb = warp + 8 * q;
    if (cb < KB) {
      double a[NBLK][CH][2];
#pragma unroll
      for (int rb = 0; rb < NBLK; ++rb)
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) a[rb][ch][0] = a[rb][ch][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < DP / 4; ++kk)
#pragma unroll
        for (int rb = 0; rb < NBLK; ++rb)
          dmma(a[rb][kk % CH][0], a[rb][kk % CH][1], Ys[rowA[rb] * LDY + 4 * kk + tig], bf[q][kk]);
#pragma unroll
      for (int rb = 0; rb < NBLK; ++rb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = cb * 8 + 2 * tig + h;
          double dot = a[rb][0][h];
#pragma unroll
          for (int ch = 1; ch < CH; ++ch) dot += a[rb][ch][h];
          const double sc = cn[c] - 2.0 * dot;
          if (sc < b1[rb] || (sc == b1[rb] && c < c1[rb])) {
            b2[rb] = b1[rb];
            b1[rb] = sc;
            c1[rb] = c;
          } else if (sc < b2[rb]) {
            b2[rb] = sc;
          }
        }
    }
  }
#pragma unroll
  for (int rb = 0; rb < NBLK; ++rb)
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {             // merge the 4 lanes of the row
      const double ob1 = __shfl_xor_sync(0xffffffffu, b1[rb], o);
      const double ob2 = __shfl_xor_sync(0xffffffffu, b2[rb], o);
      const int oc1 = __shfl_xor_sync(0xffffffffu, c1[rb], o);
      if (ob1 < b1[rb] || (ob1 == b1[rb] && oc1 < c1[rb])) {
        b2[rb] = fmin(b1[rb], ob2);
        b1[rb] = ob1;
        c1[rb] = oc1;
      } else {
        b2[rb] = fmin(b2[rb], ob1);
      }
    }
}

template <typename T, int NBW, int DP>
__global__ void __launch_bounds__(kKmThreads, NBW == 1 ? 2 : 1)
k_kmeans_step(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy, int K,
              const double* __restrict__ C, int* __restrict__ labels,
              unsigned long long* changes, double* part_inertia, double* part,
              double* __restrict__ lbound, const double* __restrict__ delta,
              const double* __restrict__ sep, double* __restrict__ ubound) {
  // DP: dim rounded up to a multiple of 16 (padding columns are zero)
  constexpr int TR = kKsRows;
  constexpr int PRE = TR * DP / kKmThreads;       // tile elements per thread
  constexpr int LDY = DP + 4;
  constexpr int KPW = 64 * NBW;
  constexpr int NST = kKsStages;                   // tile ring: 2 tiles in flight
  extern __shared__ double sm[];
  const int W = dim + 1;
  const int KB = (K + 7) / 8;
  double* Ysr = sm;                                // [NST][TR][LDY]
  double* s_lb = Ysr + NST * TR * LDY;             // [NST][TR] lower bounds of the tile rows
  double* cn = s_lb + NST * TR;                    // [KPW] ||c||^2 (inf for padding)
  double* Cs = cn + KPW;                           // [KPW][DP] centroids (direct distances)
  double* mb1 = Cs + KPW * DP;                     // [TR][8 warps]
  double* mb2 = mb1 + 8 * TR;
  int* mc1 = (int*)(mb2 + 8 * TR);                 // [TR][8 warps]
  int* tl = mc1 + 8 * TR;                          // [TR] tile labels (-1: padding row)
  int* cnt = tl + TR;                              // [KPW]
  int* fl = cnt + KPW;                             // [TR] row failed the bound test
  int* s_lab = fl + TR;                            // [NST][TR] labels of the tile rows
  __shared__ double s_in[kKmThreads / 32];
  __shared__ double s_m1, s_m2, s_cnmax;
  __shared__ int s_i1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  for (int c = tid; c < KPW; c += kKmThreads) {
    double a = 0.0;
    if (c < K)
      for (int d = 0; d < dim; ++d) a = a + C[c * dim + d] * C[c * dim + d];
    cn[c] = c < K ? a : CUDART_INF;
    cnt[c] = 0;
  }
  for (int e = tid; e < KPW * DP; e += kKmThreads) {
    const int c = e / DP, d = e % DP;
    Cs[e] = (c < K && d < dim) ? C[c * dim + d] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    // largest and second largest centroid move (excluding-own maximum), max ||c||^2
    double m1 = 0.0, m2 = 0.0, cm = 0.0;
    int i1 = -1;
    for (int c = 0; c < K; ++c) {
      cm = fmax(cm, cn[c]);
      if (!delta) continue;
      const double v = delta[c];
      if (v > m1) {
        m2 = m1;
        m1 = v;
        i1 = c;
      } else if (v > m2) {
        m2 = v;
      }
    }
    s_m1 = m1;
    s_m2 = m2;
    s_i1 = i1;
    s_cnmax = cm;
  }
  // register-resident B fragments: B[k = d][n = c] = C[c][d], d = 4 kk + tig, c = cb*8 + gid
  double bf[NBW][DP / 4];
#pragma unroll
  for (int q = 0; q < NBW; ++q) {
    const int c = (warp + 8 * q) * 8 + gid;
#pragma unroll
    for (int kk = 0; kk < DP / 4; ++kk) {
      const int d = 4 * kk + tig;
      bf[q][kk] = (c < K && d < dim) ? C[c * dim + d] : 0.0;
    }
  }
  double sacc[NBW][8][2];                          // sums S[cb*8 + j][2 lane + h]
#pragma unroll
  for (int q = 0; q < NBW; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) sacc[q][j][0] = sacc[q][j][1] = 0.0;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int rrow = tid >> 3, rw = tid & 7;         // row phases: 8 threads per row
  // tile `tile` -> ring slot: Y rows (fp64 padded; cp.async, zero-filled outside
  // [0, n) x [0, dim)), their labels and lower bounds; one commit group per call
  // full-width fp64 rows, 16-byte aligned: 16-byte copies from one base pointer
  const bool vec16 = sizeof(T) == 8 && kKmThreads % (DP / 2) == 0 && dim == DP && (ldy & 1) == 0 &&
                     (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  auto issue = [&](int64_t tile, int slot) {
    const int64_t r0 = tile * TR;
    double* Yd = Ysr + slot * TR * LDY;
    if (vec16 && r0 + TR <= n) {
      constexpr int H = DP / 2;                   // 16-byte chunks per row
      constexpr int RS = kKmThreads / H;          // rows advanced per j
      const int q0 = tid / H, c2 = 2 * (tid % H);
      const T* src = Y + (r0 + q0) * ldy + c2;
      double* dst = Yd + q0 * LDY + c2;
#pragma unroll
      for (int j = 0; j < PRE / 2; ++j) cp_async<16>(dst + j * RS * LDY, src + (int64_t)(j * RS) * ldy, 16);
    } else {
#pragma unroll
    for (int j = 0; j < PRE; ++j) {
      const int e = tid + kKmThreads * j;         // e < TR * DP
      const int q = e / DP, d = e % DP;
      const bool ok = d < dim && r0 + q < n;
      const T* src = ok ? Y + (r0 + q) * ldy + d : Y;
      if constexpr (sizeof(T) == 8) cp_async<8>(&Yd[q * LDY + d], src, ok ? 8 : 0);
      else Yd[q * LDY + d] = ok ? (double)*src : 0.0;
    }
    }
    if (tid < TR) {
      const bool ok = r0 + tid < n;
      cp_async<4>(&s_lab[slot * TR + tid], ok ? labels + r0 + tid : labels, ok ? 4 : 0);
    } else if (tid < 2 * TR && delta) {
      const bool ok = r0 + tid - TR < n;
      cp_async<8>(&s_lb[slot * TR + tid - TR], ok ? lbound + r0 + tid - TR : lbound, ok ? 8 : 0);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s0 = 0; s0 < NST - 1; ++s0) {
    const int64_t t0 = blockIdx.x + (int64_t)s0 * gridDim.x;
    if (t0 < ntiles) issue(t0, s0);
    else cp_async_commit();
  }
  __syncthreads();
  const double tau_c = s_cnmax;
  double inertia = 0.0;
  unsigned int nchg = 0, nskip = 0, ntile = 0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t r0 = tile * TR;
    const int rows = (int)imin64(TR, n - r0);
    const int slot = it % NST;
    cp_async_wait<NST - 2>();                      // this thread's copies of `tile` landed
    __syncthreads();                               // all copies visible; previous tile consumed
    {
      const int64_t nxt = tile + (int64_t)(NST - 1) * gridDim.x;
      if (nxt < ntiles) issue(nxt, (it + NST - 1) % NST);
      else cp_async_commit();
    }
    const double* Ys = Ysr + slot * TR * LDY;
    const int old_lab = rrow < rows ? s_lab[slot * TR + rrow] : -1;
    const double old_lb = delta ? s_lb[slot * TR + rrow] : 0.0;
    // ---- skip test (8 threads per row; all lanes take the shuffles)
    const bool vrow = rrow < rows;
    bool skip = false;
    double Da = 0.0, lnew = 0.0;
    {
      const int a = old_lab >= 0 ? old_lab : 0;
      double sd0 = 0.0, sd1 = 0.0;                 // ||y - c_a||^2 (padding columns are
#pragma unroll                                      // zero on both sides), two chains
      for (int i = 0; i < DP / 8; i += 2) {
        const int d = rw + 8 * i;
        const double df0 = Ys[rrow * LDY + d] - Cs[a * DP + d];
        const double df1 = Ys[rrow * LDY + d + 8] - Cs[a * DP + d + 8];
        sd0 = fma(df0, df0, sd0);
        sd1 = fma(df1, df1, sd1);
      }
      double sd = sd0 + sd1;
#pragma unroll
      for (int o = 1; o <= 4; o <<= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
      if (delta && vrow && old_lab >= 0) {
        const double dm = old_lab == s_i1 ? s_m2 : s_m1;
        Da = sd;
        lnew = old_lb - dm - kKmRel * (old_lb + dm);
        // sqrt(Da) (1 + rel) < lnew, compared in squares (Da >= 0); or Elkan's test:
        // sqrt(Da) (1 + rel) < sep[a] (half the distance from c_a to its nearest other
        // centroid, deflated) -> every other centroid is farther by the triangle inequality
        const double da2 = Da * ((1.0 + kKmRel) * (1.0 + kKmRel));
        const double sa = sep ? sep[old_lab] : 0.0;
        skip = (lnew > 0.0 && da2 < lnew * lnew) || (sa > 0.0 && da2 < sa * sa);
      }
      if (rw == 0) fl[rrow] = (vrow && !skip) ? 1 : 0;
      if (rw == 0 && skip) ++nskip;
    }
    __syncthreads();
    // products only for the rows that failed, compacted into ceil(nf / 8) blocks
    const unsigned fmask = __ballot_sync(0xffffffffu, fl[lane] != 0);   // TR == 32 rows
    const int nf = __popc(fmask);
    const int nblk = (nf + 7) >> 3;
    if (tid == 0) ntile += nblk;
    if (nblk) {
      int rowA[4];
      double b1[4], b2[4];
      int c1[4];
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        const int sl = rb * 8 + gid;                 // compact slot -> tile row
        const int rr = sl < nf ? (int)__fns(fmask, 0, sl + 1) : 0;
        rowA[rb] = rr;
        b1[rb] = CUDART_INF;
        b2[rb] = CUDART_INF;
        c1[rb] = 0x7fffffff;
      }
      switch (nblk) {
        case 1: km_assign_blocks<1, NBW, DP>(Ys, rowA, bf, cn, warp, KB, tig, b1, b2, c1); break;
        case 2: km_assign_blocks<2, NBW, DP>(Ys, rowA, bf, cn, warp, KB, tig, b1, b2, c1); break;
        case 3: km_assign_blocks<3, NBW, DP>(Ys, rowA, bf, cn, warp, KB, tig, b1, b2, c1); break;
        default: km_assign_blocks<4, NBW, DP>(Ys, rowA, bf, cn, warp, KB, tig, b1, b2, c1); break;
      }
      if (tig == 0) {
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          if (rb < nblk) {
            const int sl = rb * 8 + gid;
            mb1[sl * 8 + warp] = b1[rb];
            mb2[sl * 8 + warp] = b2[rb];
            mc1[sl * 8 + warp] = c1[rb];
          }
        }
      }
    }
    __syncthreads();
    {
      // merge across warps: 8 threads per row (thread = (row, warp slot)); when any
      // row of the tile ran the products every lane runs the butterflies, rows
      // that skipped ignore the result
      const int r = rrow, w = rw;
      int lab = old_lab;
      double dist = Da;
      double uslack = 0.0;                         // absolute error of a score-based distance
      if (fmask) {
        const bool blk = (fmask >> r) & 1u;
        const int sl = __popc(fmask & ((1u << r) - 1u));   // compact slot of row r
        double x1 = blk ? mb1[sl * 8 + w] : CUDART_INF, x2 = blk ? mb2[sl * 8 + w] : CUDART_INF;
        int xc = blk ? mc1[sl * 8 + w] : 0;
        double yn = 0.0;                           // ||y||^2: 8 partial sums, butterfly
#pragma unroll
        for (int i = 0; i < DP / 8; ++i) yn = fma(Ys[r * LDY + w + 8 * i], Ys[r * LDY + w + 8 * i], yn);
#pragma unroll
        for (int o = 1; o <= 4; o <<= 1) {
          yn += __shfl_xor_sync(0xffffffffu, yn, o);
          const double ob1 = __shfl_xor_sync(0xffffffffu, x1, o);
          const double ob2 = __shfl_xor_sync(0xffffffffu, x2, o);
          const int oc1 = __shfl_xor_sync(0xffffffffu, xc, o);
          if (ob1 < x1 || (ob1 == x1 && oc1 < xc)) {
            x2 = fmin(x1, ob2);
            x1 = ob1;
            xc = oc1;
          } else {
            x2 = fmin(x2, ob1);
          }
        }
        if (!skip && vrow) {
          // score error bound: (dim + 2) u (||y||^2 + ||c||^2) per score, dim <= 64
          const double tau = 1e-12 * (1.0 + yn + tau_c);
          lab = xc;
          dist = yn + x1;
          uslack = 2.0 * tau;
          lnew = sqrt(fmax(yn + x2 - 2.0 * tau, 0.0));
          if (!(x2 - x1 > tau)) {                  // direct form, exactly as the oracle
            double best = CUDART_INF;              // centroids c = w, w + 8, ... then merged
            int bc = 0x7fffffff;
            for (int c = w; c < K; c += 8) {
              double a = 0.0;
              for (int d = 0; d < dim; ++d) {
                const double diff = Ys[r * LDY + d] - C[c * dim + d];
                a = a + diff * diff;
              }
              if (a < best) {                      // c increases: lowest index wins ties
                best = a;
                bc = c;
              }
            }
            const unsigned gmask = 0xffu << (lane & 24);   // the row's 8 lanes (all take this branch)
#pragma unroll
            for (int o = 1; o <= 4; o <<= 1) {
              const double ob = __shfl_xor_sync(gmask, best, o);
              const int oc = __shfl_xor_sync(gmask, bc, o);
              if (ob < best || (ob == best && oc < bc)) {
                best = ob;
                bc = oc;
              }
            }
            lab = bc;
            dist = best;
            uslack = 0.0;
            lnew = 0.0;                            // near tie: recompute next step
          }
        }
      }
      if (w == 0) {
        tl[r] = r < rows ? lab : -1;
        if (r < rows) {
          if (old_lab != lab) ++nchg;
          labels[r0 + r] = lab;
          lbound[r0 + r] = lnew;
          // upper bound on the distance to the assigned centroid (the light steps'
          // Hamerly test): Da and the direct form carry <= 64 u relative error
          // (non-negative terms), a score-based distance <= 2 tau absolute
          if (ubound) ubound[r0 + r] = sqrt(fmax(dist, 0.0) + uslack) * (1.0 + kKmRel);
          inertia += dist;
          atomicAdd(&cnt[lab], 1);                 // integer: exact
        }
      }
    }
    __syncthreads();
    // ---- sums: the warp owning the label adds the row (lane: columns 2 lane, 2 lane + 1),
    // rows in tile order
    {
      const int labl = tl[lane];                     // TR == 32: lane = tile row
#pragma unroll
      for (int q = 0; q < NBW; ++q) {
        const int cb = warp + 8 * q;
        unsigned mk = __ballot_sync(0xffffffffu, (labl >> 3) == cb);
        while (mk) {
          const int r = __ffs(mk) - 1;
          mk &= mk - 1u;
          const int lab = __shfl_sync(0xffffffffu, labl, r);
          if (2 * lane < DP) {
            const double y0 = Ys[r * LDY + 2 * lane], y1 = Ys[r * LDY + 2 * lane + 1];
            switch (lab & 7) {
#define OFSC_KS_ADD(J)          \
  case J:                       \
    sacc[q][J][0] += y0;        \
    sacc[q][J][1] += y1;        \
    break;
              OFSC_KS_ADD(0) OFSC_KS_ADD(1) OFSC_KS_ADD(2) OFSC_KS_ADD(3)
              OFSC_KS_ADD(4) OFSC_KS_ADD(5) OFSC_KS_ADD(6) OFSC_KS_ADD(7)
#undef OFSC_KS_ADD
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  for (int o = 16; o; o >>= 1) {
    inertia += __shfl_xor_sync(0xffffffffu, inertia, o);
    nchg += __shfl_xor_sync(0xffffffffu, nchg, o);
    nskip += __shfl_xor_sync(0xffffffffu, nskip, o);
  }
  if (lane == 0) {
    s_in[warp] = inertia;
    if (nchg) atomicAdd(changes, (unsigned long long)nchg);        // integer: order-independent
    if (nskip) atomicAdd(changes + 1, (unsigned long long)nskip);  // statistics: rows that skipped
  }
  if (tid == 0 && ntile) atomicAdd(changes + 2, (unsigned long long)ntile);   // 8-row product blocks
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < kKmThreads / 32; ++w) a += s_in[w];
    part_inertia[blockIdx.x] = a;
  }
  double* pb = part + (int64_t)blockIdx.x * K * W;
#pragma unroll
  for (int q = 0; q < NBW; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = (warp + 8 * q) * 8 + j;
      if (c < K) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int d = 2 * lane + h;
          if (d < dim) pb[c * W + d] = sacc[q][j][h];
        }
      }
    }
  for (int c = tid; c < K; c += kKmThreads) pb[c * W + dim] = (double)cnt[c];
}

size_t kmeans_step_smem(int dim, int K) {
  const int DP = (dim + 15) & ~15;
  const int kpw = K > 64 ? 128 : 64;
  return ((size_t)kKsStages * kKsRows * (DP + 4) + kKsStages * kKsRows + kpw + (size_t)kpw * DP +
          16 * kKsRows) * 8 +
         ((size_t)10 * kKsRows + kpw + kKsStages * kKsRows) * 4;
}

bool kmeans_step_supported(int dim, int K) {
  return dim <= 64 && K <= 128 && kmeans_step_smem(dim, K) <= 200 * 1024 &&
         getenv("OFSC_KMEANS_DIRECT") == nullptr && getenv("OFSC_KMEANS_UNFUSED") == nullptr;
}

int kmeans_step_blocks(int64_t n) {
  const int64_t tiles = (n + kKsRows - 1) / kKsRows;
  const int64_t cap = (int64_t)num_sms() * 2;
  return (int)(tiles < 1 ? 1 : (tiles > cap ? cap : tiles));
}

void launch_kmeans_step(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                        const double* C, int* labels, unsigned long long* changes,
                        double* part_inertia, double* part, double* lbound, const double* delta,
                        const double* sep, double* ubound, int nblk, cudaStream_t st) {
  const size_t smem = kmeans_step_smem(dim, K);
#define OFSC_KS3(TT, NB, DPC)                                                                    \
  {                                                                                              \
    OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_step<TT, NB, DPC>,                                   \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));    \
    k_kmeans_step<TT, NB, DPC><<<nblk, kKmThreads, smem, st>>>(                                  \
        n, dim, (const TT*)Y, ldy, K, C, labels, changes, part_inertia, part, lbound, delta,    \
        sep, ubound);                                                                                  \
  }
#define OFSC_KS(TT, NB)                                                                          \
  switch ((dim + 15) / 16) {                                                                     \
    case 1: OFSC_KS3(TT, NB, 16) break;                                                          \
    case 2: OFSC_KS3(TT, NB, 32) break;                                                          \
    case 3: OFSC_KS3(TT, NB, 48) break;                                                          \
    default: OFSC_KS3(TT, NB, 64) break;                                                         \
  }
  if (dt == OFSC_F64) {
    if (K > 64) OFSC_KS(double, 2) else OFSC_KS(double, 1)
  } else {
    if (K > 64) OFSC_KS(float, 2) else OFSC_KS(float, 1)
  }
#undef OFSC_KS
#undef OFSC_KS3
  OFSC_LAUNCH_CHECK();
}

// New centroids of the fused path and their moves: one CTA per centroid,
// thread d < dim: C[c][d] = mean (empty keeps it); delta[c] = ||C_new - C_old||
// (fixed-order sum, inflated by 1e-12 so it bounds the exact move).
__global__ void k_kmeans_finish_delta(int K, int dim, const double* red, double* C,
                                      double* delta) {
  __shared__ double s[64];
  const int c = blockIdx.x, d = threadIdx.x;
  double df2 = 0.0;
  if (d < dim) {
    const double cntv = red[c * (dim + 1) + dim];
    const double old = C[c * dim + d];
    const double nw = cntv > 0.0 ? red[c * (dim + 1) + d] / cntv : old;
    C[c * dim + d] = nw;
    const double df = nw - old;
    df2 = df * df;
  }
  s[d] = df2;
  __syncthreads();
  if (d == 0) {
    double a = 0.0;
    for (int e = 0; e < dim; ++e) a += s[e];
    delta[c] = sqrt(a) * (1.0 + 1e-12);
  }
}

void launch_kmeans_finish_delta(int K, int dim, const double* red, double* C, double* delta,
                                cudaStream_t st) {
  k_kmeans_finish_delta<<<K, 64, 0, st>>>(K, dim, red, C, delta);
  OFSC_LAUNCH_CHECK();
}

// sep[c] = half the distance from centroid c to its nearest other centroid, deflated
// by 1e-12 so it bounds the exact value from below (+inf when K == 1)
__global__ void k_kmeans_halfsep(int K, int dim, const double* __restrict__ C, double* sep) {
  __shared__ double s[128];
  const int c = blockIdx.x, t = threadIdx.x;
  double best = CUDART_INF;
  for (int o = t; o < K; o += blockDim.x) {
    if (o == c) continue;
    double a = 0.0;
    for (int d = 0; d < dim; ++d) {
      const double df = C[c * dim + d] - C[o * dim + d];
      a = a + df * df;
    }
    best = fmin(best, a);
  }
  s[t] = best;
  __syncthreads();
  if (t == 0) {
    double m = CUDART_INF;
    for (int q = 0; q < (int)blockDim.x; ++q) m = fmin(m, s[q]);
    sep[c] = isinf(m) ? CUDART_INF : 0.5 * sqrt(m) * (1.0 - 1e-12);
  }
}

void launch_kmeans_halfsep(int K, int dim, const double* C, double* sep, cudaStream_t st) {
  k_kmeans_halfsep<<<K, 128, 0, st>>>(K, dim, C, sep);
  OFSC_LAUNCH_CHECK();
}

// Partial cluster sums of a contiguous row range: part[b][c][0..dim-1] = sums,
// part[b][c][dim] = count.  Thread d < dim owns column d; rows in order.
template <typename T>
__global__ void k_kmeans_partial(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy, int K,
                                 const int* __restrict__ labels, double* part) {
  extern __shared__ double acc[];          // [K][dim+1]
  const int tid = threadIdx.x;
  const int W = dim + 1;
  for (int e = tid; e < K * W; e += blockDim.x) acc[e] = 0.0;
  __syncthreads();
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per;
  const int64_t r1 = imin64(n, r0 + per);
  if (tid < W) {
    // rows in order (deterministic sums); loads of 8 rows issued ahead of the adds
    int64_t r = r0;
    for (; r + 16 <= r1; r += 16) {
      int c[16];
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) c[u] = labels[r + u];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = tid < dim ? ld1(Y + (r + u) * ldy + tid) : 1.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[c[u] * W + tid] += v[u];
    }
    for (; r < r1; ++r) {
      const int c = labels[r];
      acc[c * W + tid] += tid < dim ? ld1(Y + r * ldy + tid) : 1.0;
    }
  }
  __syncthreads();
  for (int e = tid; e < K * W; e += blockDim.x) part[(int64_t)blockIdx.x * K * W + e] = acc[e];
}

void launch_kmeans_partial(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                           const int* labels, double* part, int nblk, cudaStream_t st) {
  const size_t smem = (size_t)K * (dim + 1) * sizeof(double);
  const int th = ((dim + 1 + 31) / 32) * 32;
  if (dt == OFSC_F64) {
    OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_partial<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_kmeans_partial<double><<<nblk, th, smem, st>>>(n, dim, (const double*)Y, ldy, K, labels, part);
  } else {
    OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_partial<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_kmeans_partial<float><<<nblk, th, smem, st>>>(n, dim, (const float*)Y, ldy, K, labels, part);
  }
  OFSC_LAUNCH_CHECK();
}

// red[c][0..dim-1] = sums, red[c][dim] = count -> C[c] = mean (empty keeps C[c]).
__global__ void k_kmeans_finish(int K, int dim, const double* red, double* C) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K * dim) return;
  const int c = e / dim, d = e % dim;
  const double cnt = red[c * (dim + 1) + dim];
  if (cnt > 0.0) C[e] = red[c * (dim + 1) + d] / cnt;
}

void launch_kmeans_finish(int K, int dim, const double* red, double* C, cudaStream_t st) {
  k_kmeans_finish<<<(K * dim + 255) / 256, 256, 0, st>>>(K, dim, red, C);
  OFSC_LAUNCH_CHECK();
}


// ---------------------------------------------------------------------------
// Light Lloyd step (late steps, R28): bounds first, Y only for the rows that fail.
//   test:   u' = (u + delta[a]) (1 + rel) bounds the distance to the row's own
//           centroid from above, l' = l - max_{c != a} delta[c] - rel (l + dm) the
//           distance to every other centroid from below (Hamerly); sep[a] (half the
//           distance from c_a to its nearest other centroid, deflated) is Elkan's
//           test.  If u' < l' or u' < sep[a], every other centroid is strictly
//           farther, so Lloyd's argmin is a: the row is not read, (u', l') carried.
//   retest: a failing row is read and its exact distance Da to c_a tightens u
//           (the terms are non-negative: relative error <= (dim + 5) u << rel);
//           if now u < l' or u < sep[a] the row still keeps its label.
//   assign: otherwise the oracle's direct form (sum over d in order of
//           (y_d - C_cd)^2; this translation unit is compiled without FMA
//           contraction; ties -> lowest index) over all K centroids: one warp per
//           row, lane l owns centroids l, l + 32, ... (centroids transposed in smem:
//           conflict-free); the exact best / runner-up give the row's new (u, l).
//   sums:   only the rows whose label changed: dS[new] += y, dS[old] -= y (warp
//           owning the centroid, lane: columns 2 lane, 2 lane + 1, changed rows in
//           row order: fixed order, no atomics), dcnt by integer smem atomics;
//           part[b] = (dS, dcnt) per CTA feeds the fixed-order reduction, then
//           S += dS (k_kmeans_accum) and C = S / cnt.
// ---------------------------------------------------------------------------
constexpr int kKlPer = 4;                       // rows per thread in the bound test
constexpr int kKlRows = kKmThreads * kKlPer;    // rows per tile

template <int KPW>
__device__ __forceinline__ void kl_add(double (&sacc)[KPW][2], int j, double y0, double y1) {
#pragma unroll
  for (int q = 0; q < KPW; ++q)
    if (q == j) {
      sacc[q][0] += y0;
      sacc[q][1] += y1;
    }
}

template <typename T, int NBW>
__global__ void __launch_bounds__(kKmThreads, 2)
k_kmeans_light(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy, int K,
               const double* __restrict__ C, int* __restrict__ labels,
               double* __restrict__ ubound, double* __restrict__ lbound,
               const double* __restrict__ delta, const double* __restrict__ sep,
               unsigned long long* changes, double* part) {
  constexpr int KPW = 8 * NBW;                    // centroids owned per warp (sums)
  extern __shared__ double sm[];
  const int W = dim + 1;
  double* Ct = sm;                                // [dim][K] (transposed)
  double* yb = Ct + (size_t)K * dim;              // [8 warps][64] row buffer
  int* fl = (int*)(yb + 8 * 64);                  // [kKlRows] failing tile rows (row order)
  int* fo = fl + kKlRows;                         // [kKlRows] old label, -1: unchanged
  int* fn = fo + kKlRows;                         // [kKlRows] new label
  int* cnt = fn + kKlRows;                        // [K] count deltas
  __shared__ int s_wf[kKlPer * (kKmThreads / 32)], s_nf;
  __shared__ double s_m1, s_m2;
  __shared__ int s_i1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < K * dim; e += kKmThreads) {
    const int c = e / dim, d = e % dim;
    Ct[d * K + c] = C[e];
  }
  for (int c = tid; c < K; c += kKmThreads) cnt[c] = 0;
  if (tid == 0) {
    double m1 = 0.0, m2 = 0.0;
    int i1 = -1;
    for (int c = 0; c < K; ++c) {
      const double v = delta[c];
      if (v > m1) {
        m2 = m1;
        m1 = v;
        i1 = c;
      } else if (v > m2) {
        m2 = v;
      }
    }
    s_m1 = m1;
    s_m2 = m2;
    s_i1 = i1;
  }
  __syncthreads();
  double sacc[KPW][2];
#pragma unroll
  for (int j = 0; j < KPW; ++j) sacc[j][0] = sacc[j][1] = 0.0;
  unsigned int nchg = 0, nskip = 0;
  const int64_t ntiles = (n + kKlRows - 1) / kKlRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kKlRows;
    // tile row j * 256 + tid for j < kKlPer: loads of all four rows issued together
    bool fail[kKlPer];
    int any = 0;
#pragma unroll
    for (int j = 0; j < kKlPer; ++j) {
      const int64_t r = r0 + j * kKmThreads + tid;
      fail[j] = false;
      if (r < n) {
        const int a = labels[r];
        const double dm = a == s_i1 ? s_m2 : s_m1;
        const double ub = ubound[r], lb = lbound[r];
        const double u2 = (ub + delta[a]) * (1.0 + kKmRel);
        const double l2 = lb - dm - kKmRel * (lb + dm);
        const double sa = sep[a];
        if ((l2 > 0.0 && u2 < l2) || (sa > 0.0 && u2 < sa)) {
          ubound[r] = u2;
          lbound[r] = l2;
          ++nskip;
        } else {
          fail[j] = true;
          any = 1;
        }
      }
    }
    // failing rows compacted in row order (j, warp, lane); a tile without one costs one barrier
    unsigned bm[kKlPer];
#pragma unroll
    for (int j = 0; j < kKlPer; ++j) {
      bm[j] = __ballot_sync(0xffffffffu, fail[j]);
      if (lane == 0) s_wf[j * (kKmThreads / 32) + warp] = __popc(bm[j]);
    }
    if (__syncthreads_count(any) == 0) continue;
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kKlPer * (kKmThreads / 32); ++w) {
        const int c = s_wf[w];
        s_wf[w] = t;
        t += c;
      }
      s_nf = t;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kKlPer; ++j)
      if (fail[j])
        fl[s_wf[j * (kKmThreads / 32) + warp] + __popc(bm[j] & ((1u << lane) - 1u))] = j * kKmThreads + tid;
    __syncthreads();
    const int nf = s_nf;
    double* yr = yb + warp * 64;
    for (int q = warp; q < nf; q += kKmThreads / 32) {
      const int64_t row = r0 + fl[q];
      const int a0 = labels[row];
      double da = 0.0;                            // exact distance to the own centroid
      for (int d = lane; d < dim; d += 32) {
        const double y = ld1(Y + row * ldy + d);
        yr[d] = y;
        const double df = y - Ct[d * K + a0];
        da = fma(df, df, da);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) da += __shfl_xor_sync(0xffffffffu, da, o);
      {
        const double dm = a0 == s_i1 ? s_m2 : s_m1;
        const double lb = lbound[row];            // not yet carried: the test stored nothing
        const double l2 = lb - dm - kKmRel * (lb + dm);
        const double u2 = sqrt(da) * (1.0 + kKmRel);
        const double sa = sep[a0];
        if ((l2 > 0.0 && u2 < l2) || (sa > 0.0 && u2 < sa)) {
          if (lane == 0) {
            ubound[row] = u2;
            lbound[row] = l2;
            fo[q] = -1;
            fn[q] = a0;
            ++nskip;
          }
          __syncwarp();
          continue;
        }
      }
      __syncwarp();
      double b1 = CUDART_INF, b2 = CUDART_INF;
      int c1 = 0x7fffffff;
      auto take = [&](double a, int c) {          // c increases: lowest index wins ties
        if (a < b1) {
          b2 = b1;
          b1 = a;
          c1 = c;
        } else if (a < b2) {
          b2 = a;
        }
      };
      int c = lane;
      // centroids c and c + 32 together: two independent d-ordered chains, loads
      // unrolled ahead (each chain is the same sum, term by term, as one at a time)
      for (; c + 32 < K; c += 64) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
        for (int d = 0; d < dim; ++d) {
          const double y = yr[d];
          const double e0 = y - Ct[d * K + c], e1 = y - Ct[d * K + c + 32];
          a0 = a0 + e0 * e0;
          a1 = a1 + e1 * e1;
        }
        take(a0, c);
        take(a1, c + 32);
      }
      for (; c < K; c += 32) {
        double a = 0.0;
#pragma unroll 8
        for (int d = 0; d < dim; ++d) {
          const double diff = yr[d] - Ct[d * K + c];
          a = a + diff * diff;
        }
        take(a, c);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {             // lexicographic (distance, index) minimum
        const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
        const double ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
        const int oc1 = __shfl_xor_sync(0xffffffffu, c1, o);
        if (ob1 < b1 || (ob1 == b1 && oc1 < c1)) {
          b2 = fmin(b1, ob2);
          b1 = ob1;
          c1 = oc1;
        } else {
          b2 = fmin(b2, ob1);
        }
      }
      if (lane == 0) {
        const int old = a0;
        labels[row] = c1;
        ubound[row] = sqrt(b1) * (1.0 + kKmRel);
        lbound[row] = isinf(b2) ? CUDART_INF : sqrt(b2) * (1.0 - kKmRel);
        fo[q] = old != c1 ? old : -1;
        fn[q] = c1;
      }
      __syncwarp();
    }
    __syncthreads();
    // label changes of this tile, in row order: counts (exact) and sums (owner warps)
    for (int q = tid; q < nf; q += kKmThreads)
      if (fo[q] >= 0) {
        atomicAdd(&cnt[fn[q]], 1);
        atomicAdd(&cnt[fo[q]], -1);
        ++nchg;
      }
    for (int q = 0; q < nf; ++q) {
      const int o = fo[q];
      if (o < 0) continue;
      const int nw = fn[q];
      const bool mo = o / KPW == warp, mn = nw / KPW == warp;
      if (!mo && !mn) continue;
      double y0 = 0.0, y1 = 0.0;
      if (2 * lane < dim) {
        const T* yp = Y + (r0 + fl[q]) * ldy + 2 * lane;
        y0 = ld1(yp);
        y1 = 2 * lane + 1 < dim ? ld1(yp + 1) : 0.0;
      }
      if (mo) kl_add<KPW>(sacc, o % KPW, -y0, -y1);
      if (mn) kl_add<KPW>(sacc, nw % KPW, y0, y1);
    }
    __syncthreads();                              // fl / fo / fn reused by the next tile
  }
  for (int o = 16; o; o >>= 1) {
    nchg += __shfl_xor_sync(0xffffffffu, nchg, o);
    nskip += __shfl_xor_sync(0xffffffffu, nskip, o);
  }
  if (lane == 0) {
    if (nchg) atomicAdd(changes, (unsigned long long)nchg);        // integer: order-independent
    if (nskip) atomicAdd(changes + 1, (unsigned long long)nskip);  // statistics: rows not read
  }
  __syncthreads();
  double* pb = part + (int64_t)blockIdx.x * K * W;
#pragma unroll
  for (int j = 0; j < KPW; ++j) {
    const int c = warp * KPW + j;
    if (c < K)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int d = 2 * lane + h;
        if (d < dim) pb[c * W + d] = sacc[j][h];
      }
  }
  for (int c = tid; c < K; c += kKmThreads) pb[c * W + dim] = (double)cnt[c];
}

size_t kmeans_light_smem(int dim, int K) {
  return ((size_t)K * dim + 8 * 64) * 8 + ((size_t)3 * kKlRows + K) * 4;
}

bool kmeans_light_supported(int dim, int K) {
  const char* e = getenv("OFSC_KMEANS_LIGHT");
  return !(e && e[0] == '0') && dim <= 64 && K <= 128 && kmeans_light_smem(dim, K) <= 100 * 1024;
}

int kmeans_light_blocks(int64_t n) {
  const int64_t tiles = (n + kKlRows - 1) / kKlRows;
  const int64_t cap = (int64_t)num_sms() * 2;
  return (int)(tiles < 1 ? 1 : (tiles > cap ? cap : tiles));
}

void launch_kmeans_light(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy, int K,
                         const double* C, int* labels, double* ubound, double* lbound,
                         const double* delta, const double* sep, unsigned long long* changes,
                         double* part, int nblk, cudaStream_t st) {
  const size_t smem = kmeans_light_smem(dim, K);
#define OFSC_KL(TT, NB)                                                                            \
  {                                                                                                \
    OFSC_CUDA(cudaFuncSetAttribute(k_kmeans_light<TT, NB>,                                         \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    k_kmeans_light<TT, NB><<<nblk, kKmThreads, smem, st>>>(n, dim, (const TT*)Y, ldy, K, C, labels, \
                                                          ubound, lbound, delta, sep, changes,    \
                                                          part);                                  \
  }
  if (dt == OFSC_F64) {
    if (K > 64) OFSC_KL(double, 2) else OFSC_KL(double, 1)
  } else {
    if (K > 64) OFSC_KL(float, 2) else OFSC_KL(float, 1)
  }
#undef OFSC_KL
  OFSC_LAUNCH_CHECK();
}

// S += dS (running cluster sums and counts of the light steps)
__global__ void k_kmeans_accum(int n, double* __restrict__ S, const double* __restrict__ dS) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) S[e] += dS[e];
}

void launch_kmeans_accum(int n, double* S, const double* dS, cudaStream_t st) {
  k_kmeans_accum<<<(n + 255) / 256, 256, 0, st>>>(n, S, dS);
  OFSC_LAUNCH_CHECK();
}

// Inertia of an assignment: sum over rows of the direct-form distance to the
// row's centroid (d order, no FMA contraction); 64-row tiles staged in smem,
// one thread per row; per-CTA partial in row order -> fixed-order reduction.
template <typename T>
__global__ void __launch_bounds__(kKmThreads)
k_kmeans_inertia(int64_t n, int dim, const T* __restrict__ Y, int64_t ldy,
                 const double* __restrict__ C, const int* __restrict__ labels, double* part) {
  constexpr int TR = 64;
  __shared__ double ys[TR * 65];
  __shared__ double s_in[TR];
  const int tid = threadIdx.x;
  const int ld = dim + 1;
  double acc = 0.0;
  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TR;
    const int rows = (int)imin64(TR, n - r0);
    for (int e = tid; e < rows * dim; e += kKmThreads) {
      const int q = e / dim, d = e % dim;
      ys[q * ld + d] = ld1(Y + (r0 + q) * ldy + d);
    }
    __syncthreads();
    if (tid < rows) {
      const double* cr = C + (int64_t)labels[r0 + tid] * dim;
      double a = 0.0;
      for (int d = 0; d < dim; ++d) {
        const double diff = ys[tid * ld + d] - cr[d];
        a = a + diff * diff;
      }
      acc += a;
    }
    __syncthreads();
  }
  if (tid < TR) s_in[tid] = acc;
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int q = 0; q < TR; ++q) a += s_in[q];
    part[blockIdx.x] = a;
  }
}

void launch_kmeans_inertia(ofsc_dtype dt, int64_t n, int dim, const void* Y, int64_t ldy,
                           const double* C, const int* labels, double* part, int nblk,
                           cudaStream_t st) {
  if (dt == OFSC_F64)
    k_kmeans_inertia<double><<<nblk, kKmThreads, 0, st>>>(n, dim, (const double*)Y, ldy, C, labels, part);
  else
    k_kmeans_inertia<float><<<nblk, kKmThreads, 0, st>>>(n, dim, (const float*)Y, ldy, C, labels, part);
  OFSC_LAUNCH_CHECK();
}
}  // namespace ofsc

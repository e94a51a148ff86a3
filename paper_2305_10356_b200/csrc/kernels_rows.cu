// Row-wise kernels of the OFM iteration (Algorithm 2):
//   C3  X += alpha V, AX += alpha AV (Alg. 2 l.12, lazily applied), G = g_m(X)
//       (eq:gradientf1/g1/f2/g2) and the column dots of l.9;
//   C4  V = -G + beta Vp (Alg. 2 l.10) fused with the Grams Q = V^T V, P = V^T X
//       of the line-search cubics;
//   plus layout copies, the final update and row normalisation (Alg. 1 l.4).
// All blocks are row-major N x KP (KP = padded k, pad columns held at 0); fp32
// runs store fp32 and compute in fp64 ("fp32 policy").
#include "common.cuh"

namespace ofsc {

template <typename T>
__device__ __forceinline__ double rndT(double v) { return (double)(T)v; }

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    OFSC_CUDA(cudaGetDevice(&dev));
    OFSC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

int grid_rows(int64_t n_rows, int blocks_per_sm) {
  int64_t tiles = (n_rows + kTR - 1) / kTR;
  int64_t g = (int64_t)num_sms() * blocks_per_sm;
  if (tiles < g) g = tiles;
  return (int)(g < 1 ? 1 : g);
}

// ----------------------------------------------------------------------------
// C3: update + direction.  smem: Ms[KP][KP], Ws[KP][KP], Xs[TR][KP], AXs[TR][KP]
// ----------------------------------------------------------------------------
template <typename T, int KP, int METHOD>
__global__ void __launch_bounds__(kThreads, 2)
k_update_direction(IterParams p, int apply_update) {
  if (p.ctl->stop) return;
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;
  double* Ws = Ms + KP * KP;
  double* Xs = Ws + KP * KP;
  double* AXs = Xs + kTR * KP;
  __shared__ double s_alpha[KP];
  constexpr bool TRI = (METHOD == OFSC_TRIOFM_F1 || METHOD == OFSC_TRIOFM_F2);
  constexpr bool USE_W = (METHOD == OFSC_OFM_F2 || METHOD == OFSC_TRIOFM_F2);
  const int tid = threadIdx.x;
  for (int e = tid; e < KP * KP; e += kThreads) {
    const int j = e / KP, c = e % KP;
    const bool keep = !TRI || j <= c;              // triu keeps the diagonal (R15)
    Ms[e] = keep ? p.M[e] : 0.0;
    if (USE_W) Ws[e] = keep ? p.W[e] : 0.0;
  }
  if (tid < KP) s_alpha[tid] = apply_update ? p.alpha[tid] : 0.0;
  __syncthreads();

  T* X = (T*)p.X;
  T* AX = (T*)p.AX;
  T* G = (T*)p.G;
  const T* V = (const T*)p.V;
  const T* AV = (const T*)p.AV;
  constexpr int B = KP / 16;
  const int ti = tid >> 4, tj = tid & 15;
  double gg[B], dg[B];
#pragma unroll
  for (int j = 0; j < B; ++j) gg[j] = dg[j] = 0.0;

  const int64_t ntiles = (p.n_local + kTR - 1) / kTR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTR;
    const int rows = (int)imin64(kTR, p.n_local - row0);
    // phase A: lazily apply the previous step (Alg. 2 l.12) and stage X, AX.
    for (int e2 = tid; e2 < kTR * KP / 2; e2 += kThreads) {
      const int r = (2 * e2) / KP, c = (2 * e2) % KP;
      double2 x = make_double2(0.0, 0.0), ax = x;
      if (r < rows) {
        const int64_t off = (row0 + r) * KP + c;
        x = ld2(X + off);
        ax = ld2(AX + off);
        if (apply_update) {
          const double2 v = ld2(V + off), av = ld2(AV + off);
          x.x = rndT<T>(x.x + s_alpha[c] * v.x);
          x.y = rndT<T>(x.y + s_alpha[c + 1] * v.y);
          ax.x = rndT<T>(ax.x + s_alpha[c] * av.x);
          ax.y = rndT<T>(ax.y + s_alpha[c + 1] * av.y);
          st2(X + off, x);
          st2(AX + off, ax);
        }
      }
      Xs[r * KP + c] = x.x;
      Xs[r * KP + c + 1] = x.y;
      AXs[r * KP + c] = ax.x;
      AXs[r * KP + c + 1] = ax.y;
    }
    __syncthreads();
    // phase B: the N x k . k x k correction, 2 rows x B columns per thread.
    double sx[2][B], sa[2][B];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j = 0; j < B; ++j) sx[q][j] = sa[q][j] = 0.0;
    const int r0 = ti * 2;
    for (int j = 0; j < KP; ++j) {
      const double x0 = Xs[r0 * KP + j], x1 = Xs[(r0 + 1) * KP + j];
      double a0 = 0.0, a1 = 0.0;
      if (METHOD != OFSC_TRIOFM_F1 && METHOD != OFSC_OFM_F1) {
        a0 = AXs[r0 * KP + j];
        a1 = AXs[(r0 + 1) * KP + j];
      }
#pragma unroll
      for (int jj = 0; jj < B; ++jj) {
        const int c = jj * 16 + tj;
        const double m = Ms[j * KP + c];
        if (METHOD == OFSC_OFM_F1 || METHOD == OFSC_TRIOFM_F1) {
          sx[0][jj] = fma(x0, m, sx[0][jj]);      // X M  (or X triu(M))
          sx[1][jj] = fma(x1, m, sx[1][jj]);
        } else {
          const double w = Ws[j * KP + c];
          sx[0][jj] = fma(x0, w, sx[0][jj]);      // X W  (or X triu(W))
          sx[1][jj] = fma(x1, w, sx[1][jj]);
          sa[0][jj] = fma(a0, m, sa[0][jj]);      // AX M (or AX triu(M))
          sa[1][jj] = fma(a1, m, sa[1][jj]);
        }
      }
    }
    // phase C: G, store, column dots (G - Gp) . G and G . G
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = r0 + q;
      if (r < rows) {
#pragma unroll
        for (int jj = 0; jj < B; ++jj) {
          const int c = jj * 16 + tj;
          const double ax = AXs[r * KP + c];
          double g;
          if (METHOD == OFSC_OFM_F1) g = 4.0 * ax + 4.0 * sx[q][jj];
          else if (METHOD == OFSC_TRIOFM_F1) g = ax + sx[q][jj];
          else if (METHOD == OFSC_OFM_F2) g = 4.0 * ax - 2.0 * sx[q][jj] - 2.0 * sa[q][jj];
          else g = 2.0 * ax - sa[q][jj] - sx[q][jj];
          g = rndT<T>(g);
          const int64_t off = (row0 + r) * KP + c;
          const double gp = ld1(G + off);
          st1(G + off, g);
          gg[jj] = fma(g, g, gg[jj]);
          dg[jj] = fma(g - gp, g, dg[jj]);
        }
      }
    }
    __syncthreads();
  }
  // CTA partials: reduce the 16 row groups in fixed order.
  double* red = Xs;  // reuse (2 x 16 x KP <= 2 x TR x KP)
#pragma unroll
  for (int jj = 0; jj < B; ++jj) {
    red[ti * KP + jj * 16 + tj] = gg[jj];
    red[16 * KP + ti * KP + jj * 16 + tj] = dg[jj];
  }
  __syncthreads();
  if (tid < KP) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 16; ++q) {
      a += red[q * KP + tid];
      b += red[16 * KP + q * KP + tid];
    }
    p.part_cols[(int64_t)blockIdx.x * 2 * KP + tid] = a;
    p.part_cols[(int64_t)blockIdx.x * 2 * KP + KP + tid] = b;
  }
}

template <typename T, int KP, int METHOD>
static void launch_ud(const IterParams& p, int apply, int nblk, cudaStream_t s) {
  const size_t smem = (size_t)(2 * KP * KP + 2 * kTR * KP) * sizeof(double);
  auto kern = k_update_direction<T, KP, METHOD>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  kern<<<nblk, kThreads, smem, s>>>(p, apply);
  OFSC_LAUNCH_CHECK();
}

void launch_update_direction(ofsc_dtype dt, const IterParams& p, int apply_update, int nblk,
                             cudaStream_t s) {
  OFSC_DISPATCH_KP(p.KP, {
    if (dt == OFSC_F64) {
      switch (p.method) {
        case 0: launch_ud<double, KPC, 0>(p, apply_update, nblk, s); break;
        case 1: launch_ud<double, KPC, 1>(p, apply_update, nblk, s); break;
        case 2: launch_ud<double, KPC, 2>(p, apply_update, nblk, s); break;
        default: launch_ud<double, KPC, 3>(p, apply_update, nblk, s); break;
      }
    } else {
      switch (p.method) {
        case 0: launch_ud<float, KPC, 0>(p, apply_update, nblk, s); break;
        case 1: launch_ud<float, KPC, 1>(p, apply_update, nblk, s); break;
        case 2: launch_ud<float, KPC, 2>(p, apply_update, nblk, s); break;
        default: launch_ud<float, KPC, 3>(p, apply_update, nblk, s); break;
      }
    }
  });
}

// ----------------------------------------------------------------------------
// X += alpha V (refresh iterations and the final update)
// ----------------------------------------------------------------------------
template <typename T>
__global__ void k_update_x(IterParams p) {
  if (p.ctl->stop) return;
  T* X = (T*)p.X;
  const T* V = (const T*)p.V;
  const int64_t total = p.n_local * p.KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % p.KP);
    st1(X + e, rndT<T>(ld1(X + e) + p.alpha[c] * ld1(V + e)));
  }
}

void launch_update_x(ofsc_dtype dt, const IterParams& p, cudaStream_t s) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64) k_update_x<double><<<nb, 256, 0, s>>>(p);
  else k_update_x<float><<<nb, 256, 0, s>>>(p);
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// C4: V = -G + beta Vp, fused partial Grams Q = V^T V, P = V^T X.
// ----------------------------------------------------------------------------
template <typename T, int KP>
__global__ void __launch_bounds__(kThreads, 2) k_direction_gram(IterParams p) {
  if (p.ctl->stop) return;
  __shared__ __align__(16) double Vs[kTR * KP];
  __shared__ __align__(16) double Xs[kTR * KP];
  __shared__ double s_beta[KP];
  const int tid = threadIdx.x;
  if (tid < KP) s_beta[tid] = p.beta[tid];
  __syncthreads();
  T* V = (T*)p.V;
  const T* G = (const T*)p.G;
  const T* X = (const T*)p.X;
  const int ti = tid >> 4, tj = tid & 15;
  GramPair<KP> acc;
  acc.zero();
  const int64_t ntiles = (p.n_local + kTR - 1) / kTR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTR;
    const int rows = (int)imin64(kTR, p.n_local - row0);
    for (int e2 = tid; e2 < kTR * KP / 2; e2 += kThreads) {
      const int r = (2 * e2) / KP, c = (2 * e2) % KP;
      double2 v = make_double2(0.0, 0.0), x = v;
      if (r < rows) {
        const int64_t off = (row0 + r) * KP + c;
        const double2 g = ld2(G + off), vp = ld2(V + off);
        x = ld2(X + off);
        v.x = rndT<T>(-g.x + s_beta[c] * vp.x);
        v.y = rndT<T>(-g.y + s_beta[c + 1] * vp.y);
        st2(V + off, v);
      }
      Vs[r * KP + c] = v.x;
      Vs[r * KP + c + 1] = v.y;
      Xs[r * KP + c] = x.x;
      Xs[r * KP + c + 1] = x.y;
    }
    __syncthreads();
    acc.template accumulate<true, false>(Vs, Vs, Vs, Xs, rows, ti, tj);
    __syncthreads();
  }
  acc.store(p.part_g4 + (int64_t)blockIdx.x * 2 * KP * KP, ti, tj);
}

void launch_direction_gram(ofsc_dtype dt, const IterParams& p, int nblk, cudaStream_t s) {
  OFSC_DISPATCH_KP(p.KP, {
    if (dt == OFSC_F64) k_direction_gram<double, KPC><<<nblk, kThreads, 0, s>>>(p);
    else k_direction_gram<float, KPC><<<nblk, kThreads, 0, s>>>(p);
  });
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Generic Gram pair over local rows: part = (A^T B, A^T C)   (hook / tests)
// ----------------------------------------------------------------------------
template <typename T, int KP>
__global__ void __launch_bounds__(kThreads) k_gram_pair(int64_t n, const T* A, const T* Bm,
                                                        const T* C, double* part) {
  __shared__ __align__(16) double As[kTR * KP];
  __shared__ __align__(16) double Bs[kTR * KP];
  __shared__ __align__(16) double Cs[kTR * KP];
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  GramPair<KP> acc;
  acc.zero();
  const int64_t ntiles = (n + kTR - 1) / kTR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTR;
    const int rows = (int)imin64(kTR, n - row0);
    for (int e = tid; e < kTR * KP; e += kThreads) {
      const int r = e / KP;
      const int64_t off = row0 * KP + e;
      As[e] = r < rows ? ld1(A + off) : 0.0;
      Bs[e] = r < rows ? ld1(Bm + off) : 0.0;
      Cs[e] = r < rows ? ld1(C + off) : 0.0;
    }
    __syncthreads();
    acc.template accumulate<true, false>(As, Bs, As, Cs, rows, ti, tj);
    __syncthreads();
  }
  acc.store(part + (int64_t)blockIdx.x * 2 * KP * KP, ti, tj);
}

void launch_gram_pair(ofsc_dtype dt, int KP, int64_t n, const void* A, const void* B,
                      const void* C, double* part, int nblk, cudaStream_t st) {
  OFSC_DISPATCH_KP(KP, {
    if (dt == OFSC_F64)
      k_gram_pair<double, KPC><<<nblk, kThreads, 0, st>>>(n, (const double*)A, (const double*)B,
                                                          (const double*)C, part);
    else
      k_gram_pair<float, KPC><<<nblk, kThreads, 0, st>>>(n, (const float*)A, (const float*)B,
                                                         (const float*)C, part);
  });
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Fixed-order reduction of per-CTA partials (deterministic; no fp atomics).
// ----------------------------------------------------------------------------
__global__ void k_reduce_partials(const double* part, int nblk, int per_blk, double* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= per_blk) return;
  double a = 0.0;
  for (int b = 0; b < nblk; ++b) a += part[(int64_t)b * per_blk + g];
  out[g] = a;
}

void launch_reduce_partials(const double* part, int nblk, int per_blk, double* out,
                            cudaStream_t st) {
  k_reduce_partials<<<(per_blk + 255) / 256, 256, 0, st>>>(part, nblk, per_blk, out);
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Layout copies (user ld <-> padded KP), row normalisation.
// ----------------------------------------------------------------------------
template <typename T>
__global__ void k_copy_in(int k, int KP, int64_t n, const T* src, int64_t lds, T* dst) {
  const int64_t total = n * KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / KP;
    const int c = (int)(e % KP);
    dst[e] = c < k ? src[r * lds + c] : (T)0;
  }
}
template <typename T>
__global__ void k_copy_out(int k, int KP, int64_t n, const T* src, T* dst, int64_t ldd) {
  const int64_t total = n * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k;
    const int c = (int)(e % k);
    dst[r * ldd + c] = src[r * KP + c];
  }
}

void launch_copy_in(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, int64_t lds,
                    void* dst, cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64) k_copy_in<double><<<nb, 256, 0, st>>>(k, KP, n, (const double*)src, lds, (double*)dst);
  else k_copy_in<float><<<nb, 256, 0, st>>>(k, KP, n, (const float*)src, lds, (float*)dst);
  OFSC_LAUNCH_CHECK();
}
void launch_copy_out(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, void* dst,
                     int64_t ldd, cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64) k_copy_out<double><<<nb, 256, 0, st>>>(k, KP, n, (const double*)src, (double*)dst, ldd);
  else k_copy_out<float><<<nb, 256, 0, st>>>(k, KP, n, (const float*)src, (float*)dst, ldd);
  OFSC_LAUNCH_CHECK();
}

// y_i = x_i / ||x_i||_2 (Alg. 1 l.4); one warp per row, fp64 arithmetic.
template <typename T>
__global__ void k_row_normalize(int64_t n, int k, const T* X, int64_t ldx, T* Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    double v0 = lane < k ? ld1(X + r * ldx + lane) : 0.0;
    double v1 = lane + 32 < k ? ld1(X + r * ldx + lane + 32) : 0.0;
    double ss = v0 * v0 + v1 * v1;
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double nrm = sqrt(ss);
    if (lane < k) st1(Y + r * ldy + lane, nrm > 0.0 ? v0 / nrm : 0.0);
    if (lane + 32 < k) st1(Y + r * ldy + lane + 32, nrm > 0.0 ? v1 / nrm : 0.0);
  }
}

void launch_row_normalize(ofsc_dtype dt, int64_t n, int k, const void* X, int64_t ldx, void* Y,
                          int64_t ldy, cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64)
    k_row_normalize<double><<<nb, 256, 0, st>>>(n, k, (const double*)X, ldx, (double*)Y, ldy);
  else
    k_row_normalize<float><<<nb, 256, 0, st>>>(n, k, (const float*)X, ldx, (float*)Y, ldy);
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

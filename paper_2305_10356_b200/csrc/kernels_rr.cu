// Orthogonalisation + Rayleigh-Ritz post-step and the relerr metric
// ("one SpMM, several dot products, and an
// eigendecomposition of a k x k matrix"; P:589 relerr).
//
// Given M = X^T X and W = X^T (A X) (from the SpMM + Gram step, refresh mode):
//   k_rr_small (1 CTA):  M = L L^T (Cholesky-QR: Q = X L^{-T}, DESIGN R24);
//                        H = L^{-1} ((W + W^T)/2) L^{-T} (R25); H = Z Theta Z^T by
//                        parallel cyclic Jacobi (round-robin ordering: k/2 disjoint
//                        rotations per step); Theta ascending; Tm = L^{-T} Z.
//   k_rr_rows:           U = X Tm (Ritz vectors), A U = (A X) Tm (no second SpMM),
//                        per-CTA partials of ||A U - U Theta||_F^2 and
//                        ||U (Theta + 4)||_F^2 (B = A + 4I, R26).
#include <math_constants.h>

#include "common.cuh"

namespace ofsc {

constexpr int kRRThreads = 256;

// smem: L, H, Z as k x k row-major (ld = k); c/s per pair; flags.
__global__ void __launch_bounds__(kRRThreads) k_rr_small(const double* __restrict__ Mg,
                                                         const double* __restrict__ Wg, int KP,
                                                         int k, double* Tm, double* theta,
                                                         int* status) {
  extern __shared__ double sm[];
  double* L = sm;                 // k x k
  double* H = L + k * k;          // k x k
  double* Z = H + k * k;          // k x k
  double* cs = Z + k * k;         // [64][2]
  double* red = cs + 128;         // [kRRThreads]
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < k * k; e += kRRThreads) {
    const int i = e / k, j = e % k;
    L[e] = 0.0;
    H[e] = 0.5 * (Wg[i * KP + j] + Wg[j * KP + i]);
    Z[e] = i == j ? 1.0 : 0.0;
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  // ---- Cholesky M = L L^T (column by column)
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      double d = Mg[j * KP + j];
      for (int p = 0; p < j; ++p) d -= L[j * k + p] * L[j * k + p];
      if (!(d > 0.0) || !isfinite(d)) s_bad = 1;
      L[j * k + j] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += kRRThreads) {
      double a = Mg[i * KP + j];
      for (int p = 0; p < j; ++p) a -= L[i * k + p] * L[j * k + p];
      L[i * k + j] = a / L[j * k + j];
    }
    __syncthreads();
  }
  // ---- H <- L^{-1} H (forward substitution, one column per thread), then
  //      H <- (L^{-1} H^T)^T, i.e. L^{-1} Ws L^{-T}
  for (int pass = 0; pass < 2; ++pass) {
    for (int c = tid; c < k; c += kRRThreads) {
      for (int i = 0; i < k; ++i) {
        double a = pass == 0 ? H[i * k + c] : Z[i * k + c];
        for (int p = 0; p < i; ++p) a -= L[i * k + p] * (pass == 0 ? H[p * k + c] : Z[p * k + c]);
        if (pass == 0) H[i * k + c] = a / L[i * k + i];
        else Z[i * k + c] = a / L[i * k + i];
      }
    }
    __syncthreads();
    if (pass == 0) {   // Z <- H^T (scratch), then solve into Z
      for (int e = tid; e < k * k; e += kRRThreads) Z[e] = H[(e % k) * k + e / k];
      __syncthreads();
    }
  }
  // H = Z^T symmetrised exactly; Z <- I
  for (int e = tid; e < k * k; e += kRRThreads) {
    const int i = e / k, j = e % k;
    H[e] = 0.5 * (Z[j * k + i] + Z[i * k + j]);
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += kRRThreads) Z[e] = (e / k == e % k) ? 1.0 : 0.0;
  __syncthreads();
  // ---- parallel cyclic Jacobi (circle-method round robin over m = k rounded to even)
  const int m = (k + 1) & ~1;
  const int npairs = m / 2;
  for (int sweep = 0; sweep < 60 && k > 1; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < k * k; e += kRRThreads) {
      const double v = H[e] * H[e];
      tot += v;
      if (e / k != e % k) off += v;
    }
    red[tid] = off;
    __syncthreads();
    if (tid == 0) {
      double a = 0.0;
      for (int t = 0; t < kRRThreads; ++t) a += red[t];
      cs[0] = a;
    }
    __syncthreads();
    red[tid] = tot;
    __syncthreads();
    if (tid == 0) {
      double a = 0.0;
      for (int t = 0; t < kRRThreads; ++t) a += red[t];
      cs[1] = a;
    }
    __syncthreads();
    const bool done = sqrt(cs[0]) <= 1e-14 * fmax(1.0, sqrt(cs[1]));
    __syncthreads();
    if (done) break;
    for (int r = 0; r < m - 1; ++r) {
      // rotation parameters of the round's disjoint pairs
      for (int i = tid; i < npairs; i += kRRThreads) {
        const int a = i == 0 ? 0 : ((i - 1 + r) % (m - 1)) + 1;
        const int j2 = m - 1 - i;
        const int b = ((j2 - 1 + r) % (m - 1)) + 1;
        const int p = a < b ? a : b, q = a < b ? b : a;
        double c = 1.0, s = 0.0;
        if (q < k) {
          const double apq = H[p * k + q];
          if (apq != 0.0) {
            const double tau = (H[q * k + q] - H[p * k + p]) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[2 * i] = c;
        cs[2 * i + 1] = s;
      }
      __syncthreads();
      // columns: H <- H J, Z <- Z J
      for (int e = tid; e < npairs * k; e += kRRThreads) {
        const int i = e / k, row = e % k;
        const int a = i == 0 ? 0 : ((i - 1 + r) % (m - 1)) + 1;
        const int b = ((m - 1 - i - 1 + r) % (m - 1)) + 1;
        const int p = a < b ? a : b, q = a < b ? b : a;
        if (q >= k) continue;
        const double c = cs[2 * i], s = cs[2 * i + 1];
        const double hp = H[row * k + p], hq = H[row * k + q];
        H[row * k + p] = c * hp - s * hq;
        H[row * k + q] = s * hp + c * hq;
        const double zp = Z[row * k + p], zq = Z[row * k + q];
        Z[row * k + p] = c * zp - s * zq;
        Z[row * k + q] = s * zp + c * zq;
      }
      __syncthreads();
      // rows: H <- J^T H
      for (int e = tid; e < npairs * k; e += kRRThreads) {
        const int i = e / k, col = e % k;
        const int a = i == 0 ? 0 : ((i - 1 + r) % (m - 1)) + 1;
        const int b = ((m - 1 - i - 1 + r) % (m - 1)) + 1;
        const int p = a < b ? a : b, q = a < b ? b : a;
        if (q >= k) continue;
        const double c = cs[2 * i], s = cs[2 * i + 1];
        const double hp = H[p * k + col], hq = H[q * k + col];
        H[p * k + col] = c * hp - s * hq;
        H[q * k + col] = s * hp + c * hq;
      }
      __syncthreads();
    }
  }
  // ---- sort ascending (stable), Tm = L^{-T} Z[:, order]
  __shared__ int order[64];
  if (tid == 0) {
    for (int i = 0; i < k; ++i) order[i] = i;
    for (int i = 1; i < k; ++i) {          // insertion sort: stable
      const int o = order[i];
      const double v = H[o * k + o];
      int j = i - 1;
      while (j >= 0 && H[order[j] * k + order[j]] > v) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = o;
    }
    *status = s_bad;
  }
  __syncthreads();
  for (int c = tid; c < KP; c += kRRThreads) theta[c] = c < k ? H[order[c] * k + order[c]] : 0.0;
  for (int e = tid; e < KP * KP; e += kRRThreads) Tm[e] = 0.0;
  __syncthreads();
  for (int c = tid; c < k; c += kRRThreads) {
    const int oc = order[c];
    for (int i = k - 1; i >= 0; --i) {       // L^T upper triangular: back substitution
      double a = Z[i * k + oc];
      for (int p = i + 1; p < k; ++p) a -= L[p * k + i] * Tm[p * KP + c];
      Tm[i * KP + c] = a / L[i * k + i];
    }
  }
}

void launch_rr_small(const double* M, const double* W, int KP, int k, double* Tm, double* theta,
                     int* status, cudaStream_t st) {
  const size_t smem = ((size_t)3 * k * k + 128 + kRRThreads) * sizeof(double);
  OFSC_CUDA(cudaFuncSetAttribute(k_rr_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  k_rr_small<<<1, kRRThreads, smem, st>>>(M, W, KP, k, Tm, theta, status);
  OFSC_LAUNCH_CHECK();
}

// One warp per row; lane j owns columns j and j + 32.  part[b] = (resid^2, den^2).
template <typename T>
__global__ void __launch_bounds__(kRRThreads) k_rr_rows(int64_t n, int k, int KP, const T* X,
                                                        const T* AX, const double* Tmg,
                                                        const double* thg, T* U, double* part) {
  extern __shared__ double sm[];
  double* Tm = sm;                 // KP x KP
  double* th = Tm + KP * KP;       // KP
  __shared__ double sr[kRRThreads / 32], sd[kRRThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < KP * KP; e += kRRThreads) Tm[e] = Tmg[e];
  for (int e = tid; e < KP; e += kRRThreads) th[e] = thg[e];
  __syncthreads();
  double r2 = 0.0, d2 = 0.0;
  const int64_t nw = (int64_t)gridDim.x * (kRRThreads / 32);
  for (int64_t r = (int64_t)blockIdx.x * (kRRThreads / 32) + warp; r < n; r += nw) {
    const T* x = X + r * KP;
    const T* ax = AX + r * KP;
    double u0 = 0.0, u1 = 0.0, a0 = 0.0, a1 = 0.0;
    for (int i = 0; i < k; ++i) {
      const double xi = (double)x[i], axi = (double)ax[i];
      const double t0 = lane < KP ? Tm[i * KP + lane] : 0.0;
      const double t1 = lane + 32 < KP ? Tm[i * KP + lane + 32] : 0.0;
      u0 = fma(xi, t0, u0);
      u1 = fma(xi, t1, u1);
      a0 = fma(axi, t0, a0);
      a1 = fma(axi, t1, a1);
    }
    if (lane < k) {
      const double e = a0 - u0 * th[lane], dd = u0 * (th[lane] + 4.0);
      r2 = fma(e, e, r2);
      d2 = fma(dd, dd, d2);
    }
    if (lane + 32 < k) {
      const double e = a1 - u1 * th[lane + 32], dd = u1 * (th[lane + 32] + 4.0);
      r2 = fma(e, e, r2);
      d2 = fma(dd, dd, d2);
    }
    if (lane < KP) U[r * KP + lane] = (T)(lane < k ? u0 : 0.0);
    if (lane + 32 < KP) U[r * KP + lane + 32] = (T)(lane + 32 < k ? u1 : 0.0);
  }
  for (int o = 16; o; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    d2 += __shfl_xor_sync(0xffffffffu, d2, o);
  }
  if (lane == 0) {
    sr[warp] = r2;
    sd[warp] = d2;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kRRThreads / 32; ++w) {
      a += sr[w];
      b += sd[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

int rr_rows_blocks(int64_t n) {
  int64_t b = (n + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

void launch_rr_rows(ofsc_dtype dt, int64_t n, int k, int KP, const void* X, const void* AX,
                    const double* Tm, const double* theta, void* U, double* part, int nblk,
                    cudaStream_t st) {
  const size_t smem = ((size_t)KP * KP + KP) * sizeof(double);
  if (dt == OFSC_F64) {
    OFSC_CUDA(cudaFuncSetAttribute(k_rr_rows<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    k_rr_rows<double><<<nblk, kRRThreads, smem, st>>>(n, k, KP, (const double*)X,
                                                      (const double*)AX, Tm, theta, (double*)U,
                                                      part);
  } else {
    OFSC_CUDA(cudaFuncSetAttribute(k_rr_rows<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    k_rr_rows<float><<<nblk, kRRThreads, smem, st>>>(n, k, KP, (const float*)X,
                                                     (const float*)AX, Tm, theta, (float*)U, part);
  }
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

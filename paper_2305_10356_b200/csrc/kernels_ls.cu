// k x k stage of the iteration, on the device (no host round trip):
//   k_beta        column-wise Polak-Ribiere beta (Alg. 2 l.9), ||G||_F,
//                 objective f(X_t), convergence / divergence flags, history;
//   k_linesearch  exact line search: cubic coefficients from the
//                 Grams Q, P, T, R', M, W, real roots by Cardano / trigonometric
//                 form, 2 Newton polishes, min-psi selection, then the
//                 algebraic update M += P^T D + D P + D Q D, W += R' D + D R'^T + D T D.
// This translation unit is compiled with -fmad=false so that every scalar
// expression rounds exactly as written (R10: both sides run the
// identical root procedure).
#include <math_constants.h>

#include "common.cuh"
#include "sm100.cuh"

namespace ofsc {

// ---------------------------------------------------------------------------
// Root procedure (restated from DESIGN.md R7-R10).
// Codes: 0 zero, 1 noroot, 2 linear, 3 quad1, 4 quad2, 5 one, 6 triple,
//        7 double, 8..10 three roots (selected j), 11 diverged.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sgn1(double x) { return x < 0.0 ? -1.0 : 1.0; }
__device__ __forceinline__ double ceval(double c3, double c2, double c1, double c0, double a) {
  return ((c3 * a + c2) * a + c1) * a + c0;
}
__device__ __forceinline__ double cder(double c3, double c2, double c1, double a) {
  return (3.0 * c3 * a + 2.0 * c2) * a + c1;
}
__device__ __forceinline__ double cpsi(double c3, double c2, double c1, double c0, double a) {
  return a * (c0 + a * (0.5 * c1 + a * (c2 / 3.0 + a * (0.25 * c3))));
}
__device__ __forceinline__ double polish(double c3, double c2, double c1, double c0, double a) {
  for (int it = 0; it < 2; ++it) {
    const double d = cder(c3, c2, c1, a);
    if (d != 0.0) a = a - ceval(c3, c2, c1, c0, a) / d;
  }
  return a;
}

__device__ double select_step(double c3, double c2, double c1, double c0, int* code) {
  if (!isfinite(c3) || !isfinite(c2) || !isfinite(c1) || !isfinite(c0)) {
    *code = 11;
    return 0.0;
  }
  double roots[3];
  int nr = 0, cd = 0;
  if (c3 == 0.0 && c2 == 0.0 && c1 == 0.0 && c0 == 0.0) {
    *code = 0;
    return 0.0;
  }
  if (c3 == 0.0) {
    if (c2 == 0.0) {
      if (c1 == 0.0) {
        *code = 1;
        return 0.0;
      }
      roots[nr++] = -c0 / c1;
      cd = 2;
    } else {
      const double disc = c1 * c1 - 4.0 * c2 * c0;
      if (disc < 0.0) {
        *code = 1;
        return 0.0;
      }
      const double q = -0.5 * (c1 + sgn1(c1) * sqrt(disc));
      if (q == 0.0) {
        roots[nr++] = 0.0;
        cd = 3;
      } else {
        roots[nr++] = q / c2;
        roots[nr++] = c0 / q;
        cd = 4;
      }
    }
  } else {
    const double a = c2 / c3, b = c1 / c3, c = c0 / c3;
    const double p = b - (a * a) / 3.0;
    const double q = ((2.0 * a) * a * a) / 27.0 - (a * b) / 3.0 + c;
    const double h = q / 2.0, t = p / 3.0;
    const double D = h * h + (t * t) * t;
    if (D > 0.0) {
      const double A = -sgn1(q) * cbrt(fabs(q) / 2.0 + sqrt(D));
      const double B = A != 0.0 ? -p / (3.0 * A) : 0.0;
      roots[nr++] = A + B - a / 3.0;
      cd = 5;
    } else if (D == 0.0) {
      if (p == 0.0) {
        roots[nr++] = -a / 3.0;
        cd = 6;
      } else {
        roots[nr++] = (3.0 * q) / p - a / 3.0;
        cd = 7;
      }
    } else {
      const double r = 2.0 * sqrt(-p / 3.0);
      double arg = ((3.0 * q) / (2.0 * p)) * sqrt(-3.0 / p);
      arg = fmin(1.0, fmax(-1.0, arg));
      const double theta = acos(arg) / 3.0;
      for (int j = 0; j < 3; ++j)
        roots[nr++] = -a / 3.0 + r * cos(theta - (2.0 * CUDART_PI * (double)j) / 3.0);
      cd = 8;
    }
  }
  double best = 0.0, bpsi = 0.0;
  int bj = 0;
  for (int j = 0; j < nr; ++j) {
    const double rj = polish(c3, c2, c1, c0, roots[j]);
    const double v = cpsi(c3, c2, c1, c0, rj);
    if (j == 0 || v < bpsi ||
        (v == bpsi && (fabs(rj) < fabs(best) || (fabs(rj) == fabs(best) && rj < best)))) {
      best = rj;
      bpsi = v;
      bj = j;
    }
  }
  if (!isfinite(best)) {
    *code = 11;
    return 0.0;
  }
  *code = cd == 8 ? 8 + bj : cd;
  return best;
}

// ---------------------------------------------------------------------------
// Block reduction of NS sums in fixed order (deterministic).
// ---------------------------------------------------------------------------
template <int NS>
__device__ void block_sum(double (&v)[NS], double* red /* [NS][256] */) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < NS; ++q) red[q * 256 + tid] = v[q];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (tid < w) {
#pragma unroll
      for (int q = 0; q < NS; ++q) red[q * 256 + tid] = red[q * 256 + tid] + red[q * 256 + tid + w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NS; ++q) v[q] = red[q * 256];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// beta / convergence (1 CTA of 256 threads)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_beta(IterParams p, int nblk, int reduced) {
  __shared__ double s_gg[64], s_dg[64];
  __shared__ double red[3 * 256];
  __shared__ double s_gnorm;
  __shared__ int s_stop;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  const int tid = threadIdx.x, KP = p.KP, k = p.k;
  const int t = p.ctl->iter;
  if (tid < 4 && p.spmm_ctr) p.spmm_ctr[tid] = 0ull;   // for this iteration's SpMM
  if (reduced) {
    if (tid < KP) {
      s_gg[tid] = p.colred[tid];
      s_dg[tid] = p.colred[KP + tid];
    }
  } else {
    // column c summed by 4 threads over 4 contiguous block ranges, then in range order
    const int c = tid % KP, part = tid / KP, nparts = 256 / KP;
    const int per = (nblk + nparts - 1) / nparts;
    const int q0 = part * per, q1 = min(nblk, q0 + per);
    double a = 0.0, b = 0.0;
    if (part < nparts) {
      int q = q0;
      for (; q + 8 <= q1; q += 8) {      // 16 loads in flight, added in order
        double va[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          va[u] = p.part_cols[(int64_t)(q + u) * 2 * KP + c];
          vb[u] = p.part_cols[(int64_t)(q + u) * 2 * KP + KP + c];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a += va[u];
          b += vb[u];
        }
      }
      for (; q < q1; ++q) {
        a += p.part_cols[(int64_t)q * 2 * KP + c];
        b += p.part_cols[(int64_t)q * 2 * KP + KP + c];
      }
    }
    red[tid] = a;
    red[256 + tid] = b;
    __syncthreads();
    if (tid < KP) {
      double x = red[tid], y = red[256 + tid];
      for (int q = 1; q < nparts; ++q) {
        x += red[q * KP + tid];
        y += red[256 + q * KP + tid];
      }
      s_gg[tid] = x;
      s_dg[tid] = y;
    }
    __syncthreads();
  }
  // objective from M, W: f1 = ||A||^2 + 2 tr W + ||M||^2 ; f2 = 2 tr W - tr(M W); and tr M
  const bool f1 = (p.method == OFSC_OFM_F1 || p.method == OFSC_TRIOFM_F1);
  double v[3] = {0.0, 0.0, 0.0};
  int oi = tid / k, oj = tid % k;
  const int odi = 256 / k, odj = 256 % k;
  for (int e = tid; e < k * k; e += 256, oi += odi, oj += odj) {
    if (oj >= k) {
      oj -= k;
      ++oi;
    }
    const int i = oi, j = oj;
    const double m = p.M[i * KP + j];
    v[0] += f1 ? m * m : m * p.W[j * KP + i];
    if (i == j) {
      v[1] += p.W[i * KP + i];
      v[2] += m;
    }
  }
  block_sum<3>(v, red);
  if (tid == 0) {
    double g2 = 0.0;
    for (int c = 0; c < k; ++c) g2 += s_gg[c];
    const double gn = sqrt(g2);
    const double obj = f1 ? p.fro2 + 2.0 * v[1] + v[0] : 2.0 * v[1] - v[0];
    p.hist[(int64_t)t * 4 + 0] = obj;
    p.hist[(int64_t)t * 4 + 1] = gn;
    if (t == 0) p.ctl->gnorm0 = gn;
    p.ctl->gnorm = gn;
    p.ctl->obj = obj;
    int stop = 0;
    if (!isfinite(gn)) stop = 2;
    else if (gn == 0.0 || (p.tol > 0.0 && gn <= p.tol * p.cm * sqrt(v[2]))) stop = 1;
    s_stop = stop;
    s_gnorm = gn;
  }
  __syncthreads();
  if (s_stop) {
    if (tid < KP) p.alpha[tid] = 0.0;   // the pending step has been applied by C3
    __syncthreads();
    if (tid == 0) p.ctl->stop = s_stop;
    return;
  }
  if (tid < KP) {
    double b = 0.0;
    if (t > 0 && p.beta_rule != OFSC_BETA_ZERO && tid < k) {
      const double den = p.gg_prev[tid];
      b = den > 0.0 ? s_dg[tid] / den : 0.0;
      if (p.beta_rule == OFSC_BETA_PR_PLUS) b = fmax(b, 0.0);
    }
    p.beta[tid] = b;
    p.gg_prev[tid] = s_gg[tid];
  }
}

void launch_beta(const IterParams& p, int nblk, int reduced, cudaStream_t st) {
  launch_k(k_beta, dim3(1), dim3(256), 0, st, pdl_take(), p, nblk, reduced);
}

__global__ void k_reduce_cols(IterParams p, int nblk) {
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  const int tid = threadIdx.x;
  if (tid < 2 * p.KP) {
    double a = 0.0;
    for (int q = 0; q < nblk; ++q) a += p.part_cols[(int64_t)q * 2 * p.KP + tid];
    p.colred[tid] = a;
  }
}

void launch_reduce_cols(const IterParams& p, int nblk, cudaStream_t st) {
  k_reduce_cols<<<1, 128, 0, st>>>(p, nblk);
  OFSC_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Line search core: coefficients (eq:f1-derivative, eq:alphai-f1,
// eq:f2-derivative, eq:alphai-f2), roots, alpha, M/W update.
// [X U(Y)]_ii = sum_{j<=i} X_ij Y_ji ;  [X U(Y^T)]_ii = sum_{j<=i} X_ij Y_ij.
// ---------------------------------------------------------------------------
struct LsOut {
  int diverged, n_three, n_zero;
  double amin, amax;
};

__device__ void ls_core(int method, int k, int KP, const double* Q, const double* P,
                        const double* Tm, const double* Rp, double* M, double* W,
                        int line_search, double alpha_fixed, double* alpha, int* codes,
                        double* red, LsOut* out) {
  __shared__ double s_alpha[64];
  __shared__ int s_code[64];
  const int tid = threadIdx.x;
  const bool tri = (method == OFSC_TRIOFM_F1 || method == OFSC_TRIOFM_F2);
#define QQ(i, j) Q[(i) * KP + (j)]
#define PP(i, j) P[(i) * KP + (j)]
#define TT(i, j) Tm[(i) * KP + (j)]
#define RR(i, j) Rp[(i) * KP + (j)]
#define MM(i, j) M[(i) * KP + (j)]
#define WW(i, j) W[(i) * KP + (j)]
  if (!line_search) {
    if (tid < 64) {
      s_alpha[tid] = tid < k ? alpha_fixed : 0.0;
      s_code[tid] = 0;
    }
  } else if (!tri) {
    // whole-trace sums
    double v[11];
#pragma unroll
    for (int q = 0; q < 11; ++q) v[q] = 0.0;
    // (i, j) = (e / k, e % k) for e = tid, tid + 256, ..., stepped without divisions
    int i = tid / k, j = tid % k;
    const int di = 256 / k, dj = 256 % k;
    for (int e = tid; e < k * k; e += 256, i += di, j += dj) {
      if (j >= k) {
        j -= k;
        ++i;
      }
      const double q_ij = QQ(i, j), p_ij = PP(i, j);
      if (method == OFSC_OFM_F1) {
        v[0] += q_ij * QQ(j, i);          // tr(QQ)
        v[1] += q_ij * p_ij;              // tr(Q P^T)
        v[2] += p_ij * PP(j, i);          // tr(PP)
        v[3] += p_ij * p_ij;              // tr(P P^T)
        v[4] += q_ij * MM(j, i);          // tr(QM)
        v[5] += p_ij * MM(j, i);          // tr(PM)
        if (i == j) {
          v[6] += TT(i, i);               // tr T
          v[7] += RR(i, i);               // tr R = tr R'
        }
      } else {
        v[0] += q_ij * TT(j, i);          // tr(QT)
        v[1] += p_ij * TT(j, i);          // tr(PT)
        v[2] += q_ij * RR(i, j);          // tr(QR),  R = R'^T
        v[3] += p_ij * RR(j, i);          // tr(P R')
        v[4] += p_ij * RR(i, j);          // tr(P R)
        v[5] += q_ij * WW(j, i);          // tr(QW)
        v[6] += MM(i, j) * TT(j, i);      // tr(MT)
        v[7] += p_ij * WW(j, i);          // tr(PW)
        v[8] += MM(i, j) * RR(i, j);      // tr(MR)
        if (i == j) {
          v[9] += TT(i, i);
          v[10] += RR(i, i);
        }
      }
    }
    block_sum<11>(v, red);
    if (tid == 0) {
      double c3, c2, c1, c0;
      if (method == OFSC_OFM_F1) {        // eq:f1-derivative (printed coefficients = phi'/4, R1)
        c3 = v[0];
        c2 = 3.0 * v[1];
        c1 = v[6] + v[2] + v[3] + v[4];
        c0 = v[7] + v[5];
      } else {                            // eq:f2-derivative
        c3 = -4.0 * v[0];
        c2 = -6.0 * (v[1] + v[2]);
        c1 = 2.0 * (2.0 * v[9] - 2.0 * v[3] - 2.0 * v[4] - v[5] - v[6]);
        c0 = 2.0 * (2.0 * v[10] - v[7] - v[8]);
      }
      int code;
      const double a = select_step(c3, c2, c1, c0, &code);
      for (int c = 0; c < 64; ++c) {
        s_alpha[c] = c < k ? a : 0.0;
        s_code[c] = code;
      }
    }
  } else if (tid < k) {
    // per-column cubics: i-th diagonal entries (R2)
    const int i = tid;
    double c3 = 0.0, c2 = 0.0, c1 = 0.0, c0 = 0.0;
    if (method == OFSC_TRIOFM_F1) {       // eq:alphai-f1
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
      for (int j = 0; j <= i; ++j) {
        s0 += QQ(i, j) * QQ(j, i);        // [Q U(Q)]
        s1 += QQ(i, j) * PP(i, j);        // [Q U(P^T)]
        s2 += QQ(i, j) * PP(j, i);        // [Q U(P)]
        s3 += PP(i, j) * QQ(j, i);        // [P U(Q)]
        s4 += PP(i, j) * PP(j, i);        // [P U(P)]
        s5 += PP(i, j) * PP(i, j);        // [P U(P^T)]
        s6 += QQ(i, j) * MM(j, i);        // [Q U(M)]
        s7 += PP(i, j) * MM(j, i);        // [P U(M)]
      }
      c3 = s0;
      c2 = s1 + s2 + s3;
      c1 = TT(i, i) + s4 + s5 + s6;
      c0 = RR(i, i) + s7;
    } else {                              // eq:alphai-f2
      double a0 = 0, a1 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0;
      double d0 = 0, d1 = 0, d2 = 0, d3 = 0, d4 = 0, d5 = 0, e0 = 0, e1 = 0;
      for (int j = 0; j <= i; ++j) {
        a0 += TT(i, j) * QQ(j, i);        // [T U(Q)]
        a1 += QQ(i, j) * TT(j, i);        // [Q U(T)]
        b0 += RR(j, i) * QQ(j, i);        // [R U(Q)]    R_ij = R'_ji
        b1 += TT(i, j) * PP(i, j);        // [T U(P^T)]
        b2 += TT(i, j) * PP(j, i);        // [T U(P)]
        b3 += PP(i, j) * TT(j, i);        // [P U(T)]
        b4 += QQ(i, j) * RR(j, i);        // [Q U(R')]
        b5 += QQ(i, j) * RR(i, j);        // [Q U(R)]
        d0 += RR(j, i) * PP(i, j);        // [R U(P^T)]
        d1 += RR(j, i) * PP(j, i);        // [R U(P)]
        d2 += TT(i, j) * MM(j, i);        // [T U(M)]
        d3 += PP(i, j) * RR(j, i);        // [P U(R')]
        d4 += PP(i, j) * RR(i, j);        // [P U(R)]
        d5 += QQ(i, j) * WW(j, i);        // [Q U(W)]
        e0 += RR(j, i) * MM(j, i);        // [R U(M)]
        e1 += PP(i, j) * WW(j, i);        // [P U(W)]
      }
      c3 = -(a0 + a1);
      c2 = -(b0 + b1 + b2 + b3 + b4 + b5);
      c1 = 2.0 * TT(i, i) - (d0 + d1 + d2 + d3 + d4 + d5);
      c0 = 2.0 * RR(i, i) - (e0 + e1);
    }
    int code;
    s_alpha[i] = select_step(c3, c2, c1, c0, &code);
    s_code[i] = code;
  } else if (tid < 64) {
    s_alpha[tid] = 0.0;
    s_code[tid] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    int div = 0, n3 = 0, nz = 0;
    double amin = 0.0, amax = 0.0;
    const int ncnt = tri ? k : 1;
    for (int c = 0; c < k; ++c) {
      const double a = s_alpha[c];
      if (c == 0 || a < amin) amin = a;
      if (c == 0 || a > amax) amax = a;
    }
    for (int c = 0; c < ncnt; ++c) {
      div |= s_code[c] == 11;
      n3 += (s_code[c] >= 8 && s_code[c] <= 10);
      nz += (line_search && s_code[c] == 0);
    }
    out->diverged = div;
    out->n_three = n3;
    out->n_zero = nz;
    out->amin = amin;
    out->amax = amax;
  }
  __syncthreads();
  const int div = out->diverged;
  if (tid < KP) {
    alpha[tid] = (div || tid >= 64) ? 0.0 : s_alpha[tid];
    if (codes) codes[tid] = tid < 64 ? s_code[tid] : 0;
  }
  if (!div && M) {
    // M += P^T D + D P + D Q D ; W += R' D + D R'^T + D T D   (D = diag alpha)
    int i = tid / KP, j = tid % KP;
    const int di = 256 / KP, dj = 256 % KP;
    for (int e = tid; e < KP * KP; e += 256, i += di, j += dj) {
      if (j >= KP) {
        j -= KP;
        ++i;
      }
      const double ai = s_alpha[i], aj = s_alpha[j];
      M[e] = M[e] + PP(j, i) * aj + ai * PP(i, j) + ai * QQ(i, j) * aj;
      W[e] = W[e] + RR(i, j) * aj + ai * RR(j, i) + ai * TT(i, j) * aj;
    }
  }
#undef QQ
#undef PP
#undef TT
#undef RR
#undef MM
#undef WW
}

__global__ void __launch_bounds__(256) k_linesearch(IterParams p) {
  __shared__ double red[11 * 256];
  __shared__ LsOut out;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  const int t = p.ctl->iter;
  const int KP = p.KP;
  const double* g = p.grams;
  ls_core(p.method, p.k, KP, g, g + KP * KP, g + 2 * KP * KP, g + 3 * KP * KP, p.M, p.W,
          p.line_search, p.alpha_fixed, p.alpha, p.hist_code ? p.hist_code + (int64_t)t * KP : nullptr,
          red, &out);
  __syncthreads();
  const int tid = threadIdx.x;
  if (p.hist_alpha && tid < KP) p.hist_alpha[(int64_t)t * KP + tid] = p.alpha[tid];
  if (tid == 0) {
    p.hist[(int64_t)t * 4 + 2] = out.amin;
    p.hist[(int64_t)t * 4 + 3] = out.amax;
    p.ctl->n_three += out.n_three;
    p.ctl->n_zero += out.n_zero;
    if (out.diverged) p.ctl->stop = 2;
    else p.ctl->iter = t + 1;
  }
}

void launch_linesearch(const IterParams& p, cudaStream_t st) {
  k_linesearch<<<1, 256, 0, st>>>(p);
  OFSC_LAUNCH_CHECK();
}

// T = diag(d_T), R' = diag(d_R) as full KP x KP matrices (zero off the diagonal)
// from the reduced column dots d = [d_T | d_R] of k_gram_diag (f1 methods).
__device__ void expand_diag(const double* __restrict__ d, double* __restrict__ tr, int KP) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = w; i < KP; i += nw)                 // row i of T and of R' (no divisions)
    for (int j = lane; j < KP; j += 32) {
      tr[i * KP + j] = i == j ? d[i] : 0.0;
      tr[KP * KP + i * KP + j] = i == j ? d[KP + i] : 0.0;
    }
}

__global__ void __launch_bounds__(256) k_expand_diag(IterParams p) {
  if (p.ctl->stop) return;
  expand_diag(p.diagred, p.grams + 2 * p.KP * p.KP, p.KP);
}

void launch_expand_diag(const IterParams& p, cudaStream_t st) {
  k_expand_diag<<<1, 256, 0, st>>>(p);
  OFSC_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) k_reduce_linesearch(IterParams p, const double* __restrict__ part,
                                                           int nblk, int diag) {
  __shared__ double red[11 * 256];
  __shared__ LsOut out;
  __shared__ int s_last;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  const int KP = p.KP;
  // diag (f1 methods): the 2 KP column dots of k_gram_diag, else the full T, R'
  const int per_blk = diag ? 2 * KP : 2 * KP * KP;
  double* dst = diag ? p.diagred : p.grams + 2 * KP * KP;
  reduce_slice32(part, nblk, per_blk, dst, red);    // this CTA's 32 outputs (common.cuh)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&p.ctl->ls_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();                                   // every slice of T, R' is visible
  if (diag) {
    expand_diag(p.diagred, p.grams + 2 * KP * KP, KP);
    __syncthreads();
  }
  const int t = p.ctl->iter;
  const double* g = p.grams;
  ls_core(p.method, p.k, KP, g, g + KP * KP, g + 2 * KP * KP, g + 3 * KP * KP, p.M, p.W,
          p.line_search, p.alpha_fixed, p.alpha, p.hist_code ? p.hist_code + (int64_t)t * KP : nullptr,
          red, &out);
  __syncthreads();
  const int tid = threadIdx.x;
  if (p.hist_alpha && tid < KP) p.hist_alpha[(int64_t)t * KP + tid] = p.alpha[tid];
  if (tid == 0) {
    p.hist[(int64_t)t * 4 + 2] = out.amin;
    p.hist[(int64_t)t * 4 + 3] = out.amax;
    p.ctl->n_three += out.n_three;
    p.ctl->n_zero += out.n_zero;
    if (out.diverged) p.ctl->stop = 2;
    else p.ctl->iter = t + 1;
    p.ctl->ls_done = 0u;                             // next iteration
  }
}

void launch_reduce_linesearch(const IterParams& p, const double* part, int nblk, int diag,
                              cudaStream_t st) {
  const int per_blk = diag ? 2 * p.KP : 2 * p.KP * p.KP;
  launch_k(k_reduce_linesearch, dim3((per_blk + 31) / 32), dim3(256), 0, st, pdl_take(), p, part,
           nblk, diag);
}

__global__ void __launch_bounds__(256) k_linesearch_hook(int method, int k, int KP,
                                                         const double* g, double* M, double* W,
                                                         double* alpha, int* codes) {
  __shared__ double red[11 * 256];
  __shared__ LsOut out;
  ls_core(method, k, KP, g, g + KP * KP, g + 2 * KP * KP, g + 3 * KP * KP, M, W, 1, 0.0, alpha,
          codes, red, &out);
}

void launch_linesearch_hook(int method, int k, int KP, const double* grams, double* M, double* W,
                            double* alpha, int* codes, cudaStream_t st) {
  k_linesearch_hook<<<1, 256, 0, st>>>(method, k, KP, grams, M, W, alpha, codes);
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

// C2: the fused SpMM + Gram step (eq:spmm P:440).
//
//   Y_i = (A Z)_i = -Z_i - s_i * sum_{j in N(i)} s_j Z_j        (A = L - 2I)
//
// One warp (or a KP/2-lane group) per row gathers the neighbour rows of Z with
// 16-byte vector loads (coalesced 2*KP*sizeof(T) bytes per neighbour), summing
// in CSR (ascending column) order.  Row tiles of 32 rows are staged in shared
// memory and the epilogue accumulates per-CTA partial Grams on the fp64 tensor
// path (DmmaGram, mma.sync m8n8k4); a fixed-order reduction (kernels_rows.cu) finishes them, so
// runs are bitwise reproducible.
//   mode 0 (iteration):  T = Z^T Y, R' = X^T Y    (Z = V)
//   mode 1 (refresh):    M = Z^T Z, W = Z^T Y     (Z = X)
#include "common.cuh"
#include "sm100.cuh"

namespace ofsc {

template <typename T>
struct Acc2 {
  T x, y;
};

template <typename T, int KP, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
k_spmm_gram(int64_t n_local, int64_t own_off, const int64_t* __restrict__ row_ptr,
            const int32_t* __restrict__ col, const double* __restrict__ s,
            const float* __restrict__ s32, const T* __restrict__ Zg, const T* __restrict__ Xown,
            T* __restrict__ Y, double* __restrict__ part, const int* stop) {
  if (stop && *stop) return;
  constexpr int LD = KP + 4;                      // padded: conflict-free DMMA fragments
  extern __shared__ __align__(16) double sp_sm[];
  double* Zs = sp_sm;
  double* Ys = Zs + kTR * LD;
  double* Xs = Ys + kTR * LD;                    // mode 0 only
  constexpr int LPR = KP / 2;                    // lanes per row (2 columns per lane)
  constexpr int RPW = (32 % LPR == 0) ? 32 / LPR : 1;  // rows per warp pass
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane / LPR, l = lane % LPR;
  const bool active = sub < RPW;
  DmmaGram<KP> acc;
  acc.zero();
  const int64_t ntiles = (n_local + kTR - 1) / kTR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTR;
    const int rows = (int)imin64(kTR, n_local - row0);
    for (int r = warp * RPW + sub; r < kTR; r += (kThreads / 32) * RPW) {
      if (!active) break;
      double2 y = make_double2(0.0, 0.0), own = y, xo = y;
      if (r < rows) {
        const int64_t i = row0 + r;
        const int64_t beg = row_ptr[i], end = row_ptr[i + 1];
        const T* zc = Zg + 2 * l;
        Acc2<T> a{(T)0, (T)0};
        int64_t e = beg;
        for (; e + 8 <= end; e += 8) {
          int c[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) c[u] = __ldg(col + e + u);
          typename Vec2<T>::type z[8];
          T sv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            z[u] = __ldg(reinterpret_cast<const typename Vec2<T>::type*>(zc + (int64_t)c[u] * KP));
            if constexpr (sizeof(T) == 8) sv[u] = (T)__ldg(s + c[u]);
            else sv[u] = (T)__ldg(s32 + c[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            a.x = fma(sv[u], z[u].x, a.x);
            a.y = fma(sv[u], z[u].y, a.y);
          }
        }
        for (; e < end; ++e) {
          const int c = __ldg(col + e);
          const typename Vec2<T>::type z =
              __ldg(reinterpret_cast<const typename Vec2<T>::type*>(zc + (int64_t)c * KP));
          T sv;
          if constexpr (sizeof(T) == 8) sv = (T)__ldg(s + c);
          else sv = (T)__ldg(s32 + c);
          a.x = fma(sv, z.x, a.x);
          a.y = fma(sv, z.y, a.y);
        }
        const typename Vec2<T>::type zo =
            *reinterpret_cast<const typename Vec2<T>::type*>(Zg + (own_off + i) * KP + 2 * l);
        T si;
        if constexpr (sizeof(T) == 8) si = (T)s[own_off + i];
        else si = s32[own_off + i];
        typename Vec2<T>::type yv;
        yv.x = -zo.x - si * a.x;
        yv.y = -zo.y - si * a.y;
        *reinterpret_cast<typename Vec2<T>::type*>(Y + i * KP + 2 * l) = yv;
        y = make_double2((double)yv.x, (double)yv.y);
        own = make_double2((double)zo.x, (double)zo.y);
        if (MODE == 0) xo = ld2(Xown + i * KP + 2 * l);
      }
      Ys[r * LD + 2 * l] = y.x;
      Ys[r * LD + 2 * l + 1] = y.y;
      Zs[r * LD + 2 * l] = own.x;
      Zs[r * LD + 2 * l + 1] = own.y;
      if (MODE == 0) {
        Xs[r * LD + 2 * l] = xo.x;
        Xs[r * LD + 2 * l + 1] = xo.y;
      }
    }
    __syncthreads();
    if (part) {
      const int r4 = (rows + 3) & ~3;
      if (MODE == 0) acc.accumulate(Zs, Ys, Xs, Ys, r4, warp, lane);   // T = Z^T Y, R' = X^T Y
      else acc.accumulate(Zs, Zs, Zs, Ys, r4, warp, lane);             // M = Z^T Z, W = Z^T Y
    }
    __syncthreads();
  }
  if (part) acc.store(part + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
}

template <typename T, int KP, int MODE>
static void launch_sg(int64_t n_local, int64_t own_off, const int64_t* row_ptr, const int32_t* col,
                      const double* s, const float* s32, const void* Zg, const void* Xown, void* Y,
                      double* part, const int* stop, int nblk, cudaStream_t st) {
  const size_t smem = (size_t)(MODE == 0 ? 3 : 2) * kTR * (KP + 4) * 8;
  auto kern = k_spmm_gram<T, KP, MODE>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  kern<<<nblk, kThreads, smem, st>>>(n_local, own_off, row_ptr, col, s, s32, (const T*)Zg,
                                     (const T*)Xown, (T*)Y, part, stop);
  OFSC_LAUNCH_CHECK();
}

void launch_spmm_gram(ofsc_dtype dt, int KP, int64_t n_local, int64_t own_off,
                      const int64_t* row_ptr, const int32_t* col, const double* s,
                      const float* s32, const void* Zg, const void* Xown, void* Y, double* part,
                      int mode, const int* stop, int nblk, cudaStream_t st) {
  OFSC_DISPATCH_KP(KP, {
    if (dt == OFSC_F64) {
      if (mode == 0) launch_sg<double, KPC, 0>(n_local, own_off, row_ptr, col, s, s32, Zg, Xown, Y, part, stop, nblk, st);
      else launch_sg<double, KPC, 1>(n_local, own_off, row_ptr, col, s, s32, Zg, Xown, Y, part, stop, nblk, st);
    } else {
      if (mode == 0) launch_sg<float, KPC, 0>(n_local, own_off, row_ptr, col, s, s32, Zg, Xown, Y, part, stop, nblk, st);
      else launch_sg<float, KPC, 1>(n_local, own_off, row_ptr, col, s, s32, Zg, Xown, Y, part, stop, nblk, st);
    }
  });
}

// Plain SpMM with arbitrary leading dimensions (ABI hook ofsc_graph_apply):
// one thread per (row, column), neighbours summed in CSR order.
template <typename T>
__global__ void k_spmm_plain(int k, int64_t n_local, int64_t own_off, const int64_t* row_ptr,
                             const int32_t* col, const double* s, const float* s32, const T* Z,
                             int64_t ldz, T* Y, int64_t ldy) {
  const int64_t total = n_local * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    const int c = (int)(e % k);
    T a = 0;
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      const int j = col[q];
      const T sj = sizeof(T) == 8 ? (T)s[j] : (T)s32[j];
      a = fma(sj, Z[(int64_t)j * ldz + c], a);
    }
    const T si = sizeof(T) == 8 ? (T)s[own_off + i] : (T)s32[own_off + i];
    Y[i * ldy + c] = -Z[(own_off + i) * ldz + c] - si * a;
  }
}

void launch_spmm_plain(ofsc_dtype dt, int k, int64_t n_local, int64_t own_off,
                       const int64_t* row_ptr, const int32_t* col, const double* s,
                       const float* s32, const void* Zg, int64_t ldz, void* Y, int64_t ldy,
                       cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64)
    k_spmm_plain<double><<<nb, 256, 0, st>>>(k, n_local, own_off, row_ptr, col, s, s32,
                                             (const double*)Zg, ldz, (double*)Y, ldy);
  else
    k_spmm_plain<float><<<nb, 256, 0, st>>>(k, n_local, own_off, row_ptr, col, s, s32,
                                            (const float*)Zg, ldz, (float*)Y, ldy);
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

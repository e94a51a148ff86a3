// Device helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "internal.h"

namespace ofsc {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

// Storage rounding: the value a block of type T holds (identity for fp64).
__device__ __forceinline__ double rnd(double v, double*) { return v; }
__device__ __forceinline__ double rnd(double v, float*) { return (double)(float)v; }

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ld2(const float* p) {
  float2 f = *reinterpret_cast<const float2*>(p);
  return make_double2((double)f.x, (double)f.y);
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
__device__ __forceinline__ void st2(float* p, double2 v) {
  *reinterpret_cast<float2*>(p) = make_float2((float)v.x, (float)v.y);
}
__device__ __forceinline__ double ld1(const double* p) { return *p; }
__device__ __forceinline__ double ld1(const float* p) { return (double)*p; }
__device__ __forceinline__ void st1(double* p, double v) { *p = v; }
__device__ __forceinline__ void st1(float* p, double v) { *p = (float)v; }

// Per-thread register block of two k x k Gram products over smem tiles.
// Thread (ti, tj) = (tid >> 4, tid & 15) owns rows i = ii*16 + ti and columns
// j = jj*16 + tj (stride-16 interleave: conflict-free smem reads).
template <int KP>
struct GramPair {
  static constexpr int B = KP / 16;
  double a[B][B];
  double b[B][B];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int j = 0; j < B; ++j) a[i][j] = b[i][j] = 0.0;
  }
  // a += L1^T R1, b += L2^T R2 over `rows` rows of KP-wide smem tiles.
  template <bool LEFT_SHARED, bool RIGHT_SHARED>
  __device__ __forceinline__ void accumulate(const double* L1, const double* R1, const double* L2,
                                             const double* R2, int rows, int ti, int tj) {
    for (int r = 0; r < rows; ++r) {
      double l1[B], l2[B], r1[B], r2[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        l1[i] = L1[r * KP + i * 16 + ti];
        l2[i] = LEFT_SHARED ? l1[i] : L2[r * KP + i * 16 + ti];
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        r1[j] = R1[r * KP + j * 16 + tj];
        r2[j] = RIGHT_SHARED ? r1[j] : R2[r * KP + j * 16 + tj];
      }
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
          a[i][j] = fma(l1[i], r1[j], a[i][j]);
          b[i][j] = fma(l2[i], r2[j], b[i][j]);
        }
    }
  }
  // part[0][i][j] = a, part[1][i][j] = b
  __device__ __forceinline__ void store(double* part, int ti, int tj) const {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int ii = i * 16 + ti, jj = j * 16 + tj;
        part[ii * KP + jj] = a[i][j];
        part[KP * KP + ii * KP + jj] = b[i][j];
      }
  }
};

// Dispatch on the padded width.
#define OFSC_DISPATCH_KP(KP, ...)                       \
  switch (KP) {                                         \
    case 16: { constexpr int KPC = 16; __VA_ARGS__; } break; \
    case 32: { constexpr int KPC = 32; __VA_ARGS__; } break; \
    case 48: { constexpr int KPC = 48; __VA_ARGS__; } break; \
    case 64: { constexpr int KPC = 64; __VA_ARGS__; } break; \
    default: throw ::ofsc::Error{OFSC_ERR_ARG, "unsupported padded k"}; \
  }

}  // namespace ofsc

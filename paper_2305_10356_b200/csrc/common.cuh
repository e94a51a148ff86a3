// Device helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "internal.h"

namespace ofsc {

// Kernel launch with optional programmatic stream serialization (PDL, see sm100.cuh):
// the kernel must call pdl_wait() before reading its predecessor's outputs.
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  OFSC_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

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

// Fixed-order reduction of nblk partial arrays (part[b][g], g < per_blk) by one
// 256-thread CTA for its 32 consecutive outputs g = blockIdx.x * 32 + lane: its 8
// warps sum 8 contiguous ranges of b in order (8 loads in flight), then the 8 range
// sums are added in range order (deterministic).  seg: 256 doubles of shared memory.
__device__ __forceinline__ void reduce_slice32(const double* __restrict__ part, int nblk,
                                               int per_blk, double* __restrict__ out,
                                               double* seg) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = blockIdx.x * 32 + lane;
  const int per_seg = (nblk + 7) / 8;
  const int b0 = w * per_seg, b1 = min(nblk, b0 + per_seg);
  double a = 0.0;
  if (g < per_blk) {
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(int64_t)(b + u) * per_blk + g];
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    for (; b < b1; ++b) a += part[(int64_t)b * per_blk + g];
  }
  seg[w * 32 + lane] = a;
  __syncthreads();
  if (w == 0 && g < per_blk) {
    double t = seg[lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += seg[q * 32 + lane];
    out[g] = t;
  }
}

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

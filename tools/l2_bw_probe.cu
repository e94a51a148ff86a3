// L2 bandwidth probe (sm_100a): the ceiling of the neighbour-row gathers of the SpMM.
//   seq:    every warp streams 16-byte loads over a buffer that fits in L2 (repeated)
//   gather: 16 lanes per row gather random 512-byte rows (64 fp64) from a window of
//           W bytes (the SpMM's access pattern; W <= L2: L2-resident, W >> L2: DRAM)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw_probe tools/l2_bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void seq_read(const double2* __restrict__ a, size_t n2, int reps, double* out) {
  double s = 0;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nt = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = tid; i < n2; i += nt) {
      const double2 v = __ldg(a + i);
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// each 16-lane group gathers `per` random rows (8 in flight) of a window of `rows` rows
__global__ void gather_rows(const double* __restrict__ z, uint32_t rows, int per, double* out) {
  const int lane = threadIdx.x & 31, sub = lane >> 4, l = lane & 15;
  const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int e = 0; e < per; e += 8) {
    double2 p[8], q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = hash32(g * 2654435761u + (e + u) * 40503u + sub) % rows;
      const double2* zr = reinterpret_cast<const double2*>(z + (size_t)r * 64 + 4 * l);
      p[u] = __ldg(zr);
      q[u] = __ldg(zr + 1);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 += p[u].x; a1 += p[u].y; a2 += q[u].x; a3 += q[u].y;
    }
  }
  if (a0 + a1 + a2 + a3 == 1.2345) out[0] = a0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, L2 %d MB\n", sms, l2 >> 20);
  const size_t big = (size_t)2560 << 20;
  double* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (size_t mb : {32, 64, 96}) {
    const size_t n2 = (mb << 20) / 16;
    const int reps = 50;
    seq_read<<<sms * 8, 256>>>((const double2*)buf, n2, 2, out);
    cudaEventRecord(a);
    seq_read<<<sms * 8, 256>>>((const double2*)buf, n2, reps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("seq   window %4zu MB: %.1f GB/s\n", mb, (double)n2 * 16 * reps / ms / 1e6);
  }
  for (size_t mb : {10, 40, 80, 120, 2560}) {
    const uint32_t rows = (uint32_t)((mb << 20) / 512);
    const int per = 512;
    for (int ctas : {3, 6}) {
      const int nb = sms * ctas;
      gather_rows<<<nb, 256>>>(buf, rows, 16, out);
      cudaEventRecord(a);
      gather_rows<<<nb, 256>>>(buf, rows, per, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)nb * 256 / 16 * per * 512;
      printf("gather window %5zu MB, %d CTAs/SM: %.1f GB/s (%.2f ms for 51.2 GB)\n", mb, ctas,
             bytes / ms / 1e6, 51.2e9 / (bytes / ms));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

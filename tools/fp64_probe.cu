// Microbenchmark: fp64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1e-3 * (threadIdx.x + 1), b = 2e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// Even warps issue DMMA, odd warps DFMA: if the two pipes are separate the mixed
// kernel finishes in about the time of its larger half.
__global__ void mixed_loop(double* out, int iters_mma, int iters_fma) {
  const bool mma = ((threadIdx.x >> 5) & 1) == 0;
  double s = 0;
  if (mma) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1e-3 * (threadIdx.x + 1), b = 2e-3;
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-7);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int tpb : {256, 512, 1024}) {
    const int blocks = sms * (2048 / tpb);
    dfma_loop<<<blocks, tpb>>>(out, 16, 1.0000001, 1e-7);
    cudaEventRecord(a);
    dfma_loop<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA tpb=%d: %.2f TFLOP/s (%.1f FMA/clk/SM at %d MHz nominal)\n", tpb, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    dmma_loop<<<blocks, tpb>>>(out, 16);
    cudaEventRecord(a);
    dmma_loop<<<blocks, tpb>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 256 * 8 * iters * (double)blocks * (tpb / 32);
    printf("DMMA tpb=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", tpb, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    const int tpb = 512, blocks = sms * 4;
    float ms;
    for (int ratio : {1, 2, 4, 8, 12}) {  // DFMA warps issue ratio x the DMMA warps' instructions
      const int im = iters, ifm = iters;  // ratio 8: equal flops in both halves
      (void)ratio;
      mixed_loop<<<blocks, tpb>>>(out, 16, 16);
      cudaEventRecord(a);
      mixed_loop<<<blocks, tpb>>>(out, im, ifm * ratio);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      const double warps = (double)blocks * tpb / 32 / 2;
      const double fm = 256.0 * 8 * im * warps, ff = 32.0 * 8 * (ifm * ratio) * warps;
      printf("MIXED ratio=%d: %.3f ms, DMMA %.2f TF + DFMA %.2f TF = %.2f TF\n", ratio, ms,
             2 * fm / ms / 1e9, 2 * ff / ms / 1e9, 2 * (fm + ff) / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

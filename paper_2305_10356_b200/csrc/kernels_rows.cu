// Row-wise kernels of the OFM iteration (Algorithm 2):
//   C3  X += alpha V, AX += alpha AV (Alg. 2 l.12, lazily applied), G = g_m(X)
//       (eq:gradientf1/g1/f2/g2) and the column dots of l.9;
//   C4  V = -G + beta Vp (Alg. 2 l.10) fused with the Grams Q = V^T V, P = V^T X
//       of the line-search cubics;
//   plus layout copies, the final update and row normalisation (Alg. 1 l.4).
// All blocks are row-major N x KP (KP = padded k, pad columns held at 0); fp32
// runs store fp32 and compute in fp64 ("fp32 policy").
#include "common.cuh"
#include "sm100.cuh"

#include <chrono>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>
#include <cstring>
#include <vector>
#include <cstdio>
#include <cstdlib>

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

// OFSC_TRACE=1: host-side phase timestamps (stream synchronised at each point)
// to stderr.  OFSC_TRACE=2: no synchronisation; each point records the host
// time and a CUDA event on `st`, and a point named "...: end" prints the list
// (host ms and device ms since the first point of the list).
void trace_point(const char* what, cudaStream_t st) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("OFSC_TRACE");
    on = (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
  }
  if (!on) return;
  static std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  if (on == 1) {
    cudaStreamSynchronize(st);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[ofsc trace] %10.2f ms  %s\n", ms, what);
    return;
  }
  struct Pt {
    const char* what;
    double host_ms;
    cudaEvent_t ev;
    double reserved_gb, used_gb;   // default mempool
  };
  static std::vector<Pt> pts;
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, st);
  double rg = 0.0, ug = 0.0;
  {
    int dev = 0;
    cudaMemPool_t pool;
    uint64_t r = 0, u = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u);
    }
    rg = r / 1e9;
    ug = u / 1e9;
  }
  pts.push_back({what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), ev, rg, ug});
  const size_t L = strlen(what);
  if (L >= 5 && strcmp(what + L - 5, ": end") == 0) {
    cudaEventSynchronize(ev);
    for (auto& p : pts) {
      float d = 0.f;
      cudaEventElapsedTime(&d, pts[0].ev, p.ev);
      fprintf(stderr, "[ofsc trace2] host %9.2f  device %9.2f ms  pool %6.2f/%6.2f GB  %s\n",
              p.host_ms - pts[0].host_ms, d, p.used_gb, p.reserved_gb, p.what);
    }
    for (auto& p : pts) cudaEventDestroy(p.ev);
    pts.clear();
  }
}

// The graph build allocates its sort / scan scratch from the device's default
// stream-ordered pool.  With the default release threshold (0) every
// synchronisation hands the freed GBs back to the driver and the next build
// maps them again (measured: 0.3-2.7 s build-time jitter at c4); keep them.
void keep_pool() {
  static unsigned long long done = 0;   // one bit per device
  int dev = 0;
  OFSC_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && (done >> dev) & 1ull) return;
  cudaMemPool_t pool;
  OFSC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~0ull;
  OFSC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  if (dev < 64) done |= 1ull << dev;
}

// Exact-size block cache on top of the pool.  Repeated calls with the same shapes
// (e.g. ofsc_spectral_cluster in a loop) get their buffers back without a pool
// round trip: with other large allocations resident, cudaMallocAsync was seen to
// block the host for 100-800 ms on some calls (bench.py e2e, OFSC_TRACE=2).
// A block freed stream-ordered (dev_free_async) is reused only on that stream;
// one freed with no queued user left (dev_free) on any stream.
namespace {
struct BlockCache {
  std::mutex m;
  std::map<std::tuple<int, size_t, cudaStream_t>, std::vector<void*>> free_blocks;
  std::unordered_map<void*, std::pair<int, size_t>> owned;   // ptr -> (device, bytes)
  size_t cached = 0;
  size_t cap = [] {                                            // bytes kept in the cache
    const char* e = getenv("OFSC_BLOCK_CACHE_GB");               // default 40 GB
    return (size_t)((e && *e) ? atof(e) : 40.0) << 30;
  }();
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();   // process lifetime (freed memory stays cached)
  return *c;
}
void* cache_take(BlockCache& c, int dev, size_t bytes, cudaStream_t key) {
  auto it = c.free_blocks.find(std::make_tuple(dev, bytes, key));
  if (it == c.free_blocks.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  c.cached -= bytes;
  return p;
}
void cache_put(void* p, cudaStream_t key, cudaStream_t free_st) {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.m);
  auto it = c.owned.find(p);
  if (it == c.owned.end()) {   // not ours (plain pool allocation)
    cudaFreeAsync(p, free_st);
    return;
  }
  const int dev = it->second.first;
  const size_t bytes = it->second.second;
  if (c.cached + bytes > c.cap) {
    c.owned.erase(it);
    cudaFreeAsync(p, free_st);
    return;
  }
  c.free_blocks[std::make_tuple(dev, bytes, key)].push_back(p);
  c.cached += bytes;
}
}  // namespace

void dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  keep_pool();
  int dev = 0;
  OFSC_CUDA(cudaGetDevice(&dev));
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> lk(c.m);
    void* q = cache_take(c, dev, bytes, nullptr);
    if (!q) q = cache_take(c, dev, bytes, st);
    if (q) {
      *p = q;
      return;
    }
  }
  cudaError_t e = cudaMallocAsync(p, bytes, st);
  if (e == cudaErrorMemoryAllocation) {
    // out of memory: hand every cached block of this device back, then retry once
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(c.m);
    for (auto& kv : c.free_blocks) {
      if (std::get<0>(kv.first) != dev) continue;
      for (void* q : kv.second) {
        cudaFreeAsync(q, std::get<2>(kv.first));
        c.owned.erase(q);
        c.cached -= std::get<1>(kv.first);
      }
      kv.second.clear();
    }
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, st);
  }
  OFSC_CUDA(e);
  std::lock_guard<std::mutex> lk(c.m);
  c.owned[*p] = std::make_pair(dev, bytes);
}

void dev_free(void* p) {
  if (p) cache_put(p, nullptr, 0);
}

void dev_trim() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaDeviceSynchronize();
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> lk(c.m);
    for (auto& kv : c.free_blocks) {
      if (std::get<0>(kv.first) != dev) continue;
      for (void* q : kv.second) {
        cudaFreeAsync(q, std::get<2>(kv.first));
        c.owned.erase(q);
        c.cached -= std::get<1>(kv.first);
      }
      kv.second.clear();
    }
  }
  cudaDeviceSynchronize();
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
}

void dev_free_async(void* p, cudaStream_t st) {
  if (p) cache_put(p, st, st);
}

int grid_rows(int64_t n_rows, int blocks_per_sm) {
  int64_t tiles = (n_rows + kTR - 1) / kTR;
  int64_t g = (int64_t)num_sms() * blocks_per_sm;
  if (tiles < g) g = tiles;
  return (int)(g < 1 ? 1 : g);
}

// ----------------------------------------------------------------------------
// X += alpha V (refresh iterations and the final update)
// ----------------------------------------------------------------------------
template <typename T>
__global__ void k_update_x(IterParams p) {
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  T* X = (T*)p.X;
  const T* V = (const T*)p.V;
  const int64_t total = p.n_local * p.KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % p.KP);
    st1(X + e, rndT<T>(fma(p.alpha[c], ld1(V + e), ld1(X + e))));   // as C3 phase A
  }
}

static thread_local bool t_pdl = false;
void pdl_next(bool on) {
  static const bool enabled = [] {
    const char* e = getenv("OFSC_PDL");
    return !(e && e[0] == '0');
  }();
  t_pdl = on && enabled;
}
bool pdl_take() {
  const bool v = t_pdl;
  t_pdl = false;
  return v;
}

void launch_update_x(ofsc_dtype dt, const IterParams& p, cudaStream_t s) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64) k_update_x<double><<<nb, 256, 0, s>>>(p);
  else k_update_x<float><<<nb, 256, 0, s>>>(p);
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Generic Gram pair over local rows: part = (A^T B, A^T C)   (hook / tests)
// ----------------------------------------------------------------------------
template <typename T, int KP>
__global__ void __launch_bounds__(kThreads) k_gram_pair(int64_t n, const T* A, const T* Bm,
                                                        const T* C, double* part) {
  constexpr int LD = KP + 4;
  extern __shared__ __align__(16) double gp_sm[];
  double* As = gp_sm;
  double* Bs = As + kTR * LD;
  double* Cs = Bs + kTR * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  typename GramSel<KP>::type acc;   // A^T A symmetric
  acc.zero();
  const int64_t ntiles = (n + kTR - 1) / kTR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTR;
    const int rows = (int)imin64(kTR, n - row0);
    for (int e = tid; e < kTR * KP; e += kThreads) {
      const int r = e / KP, c = e % KP;
      const int64_t off = row0 * KP + e;
      As[r * LD + c] = r < rows ? ld1(A + off) : 0.0;
      Bs[r * LD + c] = r < rows ? ld1(Bm + off) : 0.0;
      Cs[r * LD + c] = r < rows ? ld1(C + off) : 0.0;
    }
    __syncthreads();
    acc.accumulate(As, Bs, As, Cs, (rows + 3) & ~3, warp, lane);
    __syncthreads();
  }
  acc.store(part + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
}

void launch_gram_pair(ofsc_dtype dt, int KP, int64_t n, const void* A, const void* B,
                      const void* C, double* part, int nblk, cudaStream_t st) {
  OFSC_DISPATCH_KP(KP, {
    const size_t smem = (size_t)3 * kTR * (KPC + 4) * 8;
    if (dt == OFSC_F64) {
      OFSC_CUDA(cudaFuncSetAttribute(k_gram_pair<double, KPC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_gram_pair<double, KPC><<<nblk, kThreads, smem, st>>>(n, (const double*)A, (const double*)B,
                                                             (const double*)C, part);
    } else {
      OFSC_CUDA(cudaFuncSetAttribute(k_gram_pair<float, KPC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_gram_pair<float, KPC><<<nblk, kThreads, smem, st>>>(n, (const float*)A, (const float*)B,
                                                            (const float*)C, part);
    }
  });
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Fixed-order reduction of per-CTA partials (deterministic; no fp atomics).
// ----------------------------------------------------------------------------
// Fixed-order reduction of nblk partial arrays (reduce_slice32, common.cuh).
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ part, int nblk,
                                                         int per_blk, double* __restrict__ out) {
  __shared__ double seg[256];
  reduce_slice32(part, nblk, per_blk, out, seg);
}

void launch_reduce_partials(const double* part, int nblk, int per_blk, double* out,
                            cudaStream_t st) {
  k_reduce_partials<<<(per_blk + 31) / 32, 256, 0, st>>>(part, nblk, per_blk, out);
  OFSC_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Layout copies (user ld <-> padded KP), row normalisation.
// ----------------------------------------------------------------------------
template <typename T>
__global__ void k_copy_in(int k, int KP, int64_t n, const T* src, int64_t lds, T* dst,
                          const int32_t* perm) {
  const int64_t total = n * KP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / KP;
    const int c = (int)(e % KP);
    const int64_t u = perm ? (int64_t)perm[r] : r;
    dst[e] = c < k ? src[u * lds + c] : (T)0;
  }
}
template <typename T>
__global__ void k_copy_out(int k, int KP, int64_t n, const T* src, T* dst, int64_t ldd,
                           const int32_t* perm) {
  const int64_t total = n * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k;
    const int c = (int)(e % k);
    const int64_t u = perm ? (int64_t)perm[r] : r;
    dst[u * ldd + c] = src[r * KP + c];
  }
}

void launch_copy_in(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, int64_t lds,
                    void* dst, const int32_t* perm, cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64)
    k_copy_in<double><<<nb, 256, 0, st>>>(k, KP, n, (const double*)src, lds, (double*)dst, perm);
  else k_copy_in<float><<<nb, 256, 0, st>>>(k, KP, n, (const float*)src, lds, (float*)dst, perm);
  OFSC_LAUNCH_CHECK();
}
void launch_copy_out(ofsc_dtype dt, int k, int KP, int64_t n, const void* src, void* dst,
                     int64_t ldd, const int32_t* perm, cudaStream_t st) {
  const int nb = num_sms() * 8;
  if (dt == OFSC_F64)
    k_copy_out<double><<<nb, 256, 0, st>>>(k, KP, n, (const double*)src, (double*)dst, ldd, perm);
  else k_copy_out<float><<<nb, 256, 0, st>>>(k, KP, n, (const float*)src, (float*)dst, ldd, perm);
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

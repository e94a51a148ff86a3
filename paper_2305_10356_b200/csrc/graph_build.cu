// C1: undirected edge list -> CSR pattern of S and s = D^{-1/2} (Alg. 1 l.2).
//   1. key = (min(u,v) << 32) | max(u,v); self-loops -> sentinel (dropped, P:31 S is 0/1)
//   2. radix sort + unique: the canonical undirected edge set (duplicates collapsed)
//   3. symmetrise: (u,v) and (v,u) as (row << 32) | col, radix sort -> CSR order,
//      columns ascending within each row
//   4. degree histogram (integer atomics), exclusive scan -> row_ptr
//   5. s_i = 1 / sqrt(d_i) (0 for an isolated node), ||A||_F^2 = n + sum (s_i s_j)^2
// cub (CUDA toolkit) supplies the radix sort / unique / scan building blocks.
#include <cub/cub.cuh>

#include <algorithm>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ofsc {

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  explicit DevBuf(size_t count, cudaStream_t st) : n(count), s(st) {
    if (count) dev_alloc((void**)&p, count * sizeof(T), st);
  }
  ~DevBuf() { dev_free_async(p, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

constexpr unsigned long long kSentinel = ~0ull;

__global__ void k_make_keys(int64_t m, int64_t n, const int64_t* src, const int64_t* dst,
                            unsigned long long* keys, unsigned long long* n_loops, int* bad) {
  unsigned long long loops = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = src[e], v = dst[e];
    if (u < 0 || v < 0 || u >= n || v >= n) {
      *bad = 1;
      keys[e] = kSentinel;
      continue;
    }
    if (u == v) {
      ++loops;
      keys[e] = kSentinel;
      continue;
    }
    const unsigned long long a = (unsigned long long)(u < v ? u : v);
    const unsigned long long b = (unsigned long long)(u < v ? v : u);
    keys[e] = (a << 32) | b;
  }
  if (loops) atomicAdd(n_loops, loops);
}

__global__ void k_symmetrise(int64_t E, const unsigned long long* ukeys, unsigned long long* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ukeys[e];
    const unsigned long long u = k >> 32, v = k & 0xffffffffull;
    out[2 * e] = k;
    out[2 * e + 1] = (v << 32) | u;
  }
}

__global__ void k_split_keys(int64_t nnz, const unsigned long long* keys, int32_t* col,
                             int* deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[e];
    col[e] = (int32_t)(k & 0xffffffffull);
    atomicAdd(deg + (k >> 32), 1);
  }
}

__global__ void k_scale(int64_t n, const int* deg, double* s, int64_t* row_ptr_last,
                        unsigned long long* n_iso, int* max_deg, int64_t nnz) {
  unsigned long long iso = 0;
  int md = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = deg[i];
    s[i] = d > 0 ? 1.0 / sqrt((double)d) : 0.0;   // D^{-1/2}; isolated -> 0 (R12)
    iso += d == 0;
    md = d > md ? d : md;
  }
  if (iso) atomicAdd(n_iso, iso);
  atomicMax(max_deg, md);
  if (blockIdx.x == 0 && threadIdx.x == 0) *row_ptr_last = nnz;
}

__global__ void k_deg_to_i64(int64_t n, const int* deg, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = deg[i];
}

// per-CTA partial of sum_i sum_{j in N(i)} (s_i s_j)^2 over a contiguous row range
__global__ void k_fro2(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* s,
                       double* part) {
  __shared__ double red[256];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = imin64(n, r0 + per);
  double a = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double si2 = s[i] * s[i];
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      const double sj = s[col[q]];
      a += si2 * (sj * sj);
    }
  }
  red[threadIdx.x] = a;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

void build_csr(int64_t n, int64_t m, const int64_t* d_src, const int64_t* d_dst, CsrDevice& out,
               cudaStream_t st) {
  OFSC_REQUIRE(n >= 1 && n < (int64_t(1) << 31), OFSC_ERR_ARG, "need 1 <= n < 2^31");
  keep_pool();
  out.n = n;
  trace_point("build_csr: start", st);
  DevBuf<unsigned long long> counters(2, st);   // [0] loops, [1] isolated
  DevBuf<int> flags(2, st);                     // [0] bad endpoint, [1] max degree
  OFSC_CUDA(cudaMemsetAsync(counters.p, 0, 2 * sizeof(unsigned long long), st));
  OFSC_CUDA(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), st));
  int64_t E = 0;
  DevBuf<unsigned long long> ukeys(m > 0 ? m : 1, st);
  if (m > 0) {
    DevBuf<unsigned long long> keys(m, st);
    k_make_keys<<<blocks_for(m), 256, 0, st>>>(m, n, d_src, d_dst, keys.p, counters.p, flags.p);
    OFSC_LAUNCH_CHECK();
    DevBuf<unsigned long long> sorted(m, st);
    size_t tmp_bytes = 0;
    OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, m, 0, 64, st));
    {
      DevBuf<char> tmp(tmp_bytes, st);
      OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, m, 0, 64, st));
    }
    trace_point("build_csr: keys sorted", st);
    DevBuf<int64_t> nsel(1, st);
    tmp_bytes = 0;
    OFSC_CUDA(cub::DeviceSelect::Unique(nullptr, tmp_bytes, sorted.p, ukeys.p, nsel.p, m, st));
    {
      DevBuf<char> tmp(tmp_bytes, st);
      OFSC_CUDA(cub::DeviceSelect::Unique(tmp.p, tmp_bytes, sorted.p, ukeys.p, nsel.p, m, st));
    }
    int64_t h_nsel = 0;
    unsigned long long h_cnt[2];
    int h_flags[2];
    OFSC_CUDA(cudaMemcpyAsync(&h_nsel, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(h_cnt, counters.p, sizeof(h_cnt), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(h_flags, flags.p, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaStreamSynchronize(st));
    OFSC_REQUIRE(!h_flags[0], OFSC_ERR_RANGE, "edge endpoint outside [0, n)");
    out.n_loops = (int64_t)h_cnt[0];
    unsigned long long last = 0;
    if (h_nsel > 0)
      OFSC_CUDA(cudaMemcpy(&last, ukeys.p + h_nsel - 1, sizeof(last), cudaMemcpyDeviceToHost));
    E = h_nsel - ((h_nsel > 0 && last == kSentinel) ? 1 : 0);
  }
  trace_point("build_csr: unique", st);
  out.m_kept = E;
  out.n_dups = m - out.n_loops - E;
  out.nnz = 2 * E;
  OFSC_REQUIRE(out.nnz < (int64_t(1) << 40), OFSC_ERR_ARG, "graph too large");
  dev_alloc((void**)&out.row_ptr, (n + 1) * sizeof(int64_t), st);
  dev_alloc((void**)&out.col, (out.nnz > 0 ? out.nnz : 1) * sizeof(int32_t), st);
  dev_alloc((void**)&out.s, n * sizeof(double), st);
  DevBuf<int> deg(n, st);
  OFSC_CUDA(cudaMemsetAsync(deg.p, 0, n * sizeof(int), st));
  if (E > 0) {
    DevBuf<unsigned long long> sym(out.nnz, st), sym_sorted(out.nnz, st);
    k_symmetrise<<<blocks_for(E), 256, 0, st>>>(E, ukeys.p, sym.p);
    OFSC_LAUNCH_CHECK();
    int hi = 1;
    while ((int64_t(1) << hi) < n) ++hi;
    size_t tmp_bytes = 0;
    OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, sym.p, sym_sorted.p, out.nnz, 0,
                                             32 + hi, st));
    {
      DevBuf<char> tmp(tmp_bytes, st);
      OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, sym.p, sym_sorted.p, out.nnz, 0,
                                               32 + hi, st));
    }
    k_split_keys<<<blocks_for(out.nnz), 256, 0, st>>>(out.nnz, sym_sorted.p, out.col, deg.p);
    OFSC_LAUNCH_CHECK();
    trace_point("build_csr: symmetrised + sorted", st);
  }
  {
    DevBuf<int64_t> deg64(n, st);
    k_deg_to_i64<<<blocks_for(n), 256, 0, st>>>(n, deg.p, deg64.p);
    OFSC_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    OFSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg64.p, out.row_ptr, n, st));
    DevBuf<char> tmp(tmp_bytes, st);
    OFSC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, deg64.p, out.row_ptr, n, st));
  }
  k_scale<<<blocks_for(n), 256, 0, st>>>(n, deg.p, out.s, out.row_ptr + n, counters.p + 1,
                                         flags.p + 1, out.nnz);
  OFSC_LAUNCH_CHECK();
  const int nb = blocks_for(n) < 1024 ? blocks_for(n) : 1024;
  DevBuf<double> part(nb, st);
  k_fro2<<<nb, 256, 0, st>>>(n, out.row_ptr, out.col, out.s, part.p);
  OFSC_LAUNCH_CHECK();
  std::vector<double> hp(nb);
  unsigned long long iso = 0;
  int md = 0;
  OFSC_CUDA(cudaMemcpyAsync(hp.data(), part.p, nb * sizeof(double), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&iso, counters.p + 1, sizeof(iso), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&md, flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
  double f = 0.0;
  for (int b = 0; b < nb; ++b) f += hp[b];
  out.fro2 = (double)n + f;
  out.n_isolated = (int64_t)iso;
  out.max_deg = md;
  trace_point("build_csr: scan, s, fro2 done", st);
}

// ---- incremental CSR merge (streaming snapshots) --------
// Appends a batch of undirected edges to an existing CSR so that the result is
// exactly the CSR build_csr would produce from the concatenated edge list:
//   1. batch keys (canonical, loops -> sentinel), radix sort + unique;
//   2. symmetrise, sort by (row, col);
//   3. drop keys already present in the old CSR (binary search in the row);
//   4. new degrees = old + added, exclusive scan -> new row_ptr;
//   5. merge: one warp per row, each old / added column goes to its rank in the
//      union (binary search in the other sorted list) -> columns ascending;
//   6. s = D^{-1/2} and ||A||_F^2 recomputed by the same kernels as build_csr.
namespace {

__global__ void k_exists(int64_t nnz, const unsigned long long* keys, const int64_t* row_ptr,
                         const int32_t* col, int* keep) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[e];
    const int64_t u = (int64_t)(k >> 32);
    const int32_t v = (int32_t)(k & 0xffffffffull);
    int64_t lo = row_ptr[u], hi = row_ptr[u + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    keep[e] = (lo < row_ptr[u + 1] && col[lo] == v) ? 0 : 1;
  }
}

__global__ void k_old_degree(int64_t n, const int64_t* row_ptr, int* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = (int)(row_ptr[i + 1] - row_ptr[i]);
}

__global__ void k_add_degree(int64_t nadd, const unsigned long long* keys, int* deg_add) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nadd;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg_add + (keys[e] >> 32), 1);
}

__global__ void k_sum_deg(int64_t n, const int* a, const int* b, int* out, int64_t* out64) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = a[i] + b[i];
    out64[i] = a[i] + b[i];
  }
}

// rank of x in the sorted list p[0..len): number of elements < x
__device__ __forceinline__ int64_t rank_lt(const int32_t* p, int64_t len, int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (p[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_merge_rows(int64_t n, const int64_t* old_ptr, const int32_t* old_col,
                             const int64_t* add_ptr, const int32_t* add_col,
                             const int64_t* new_ptr, int32_t* new_col) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < n; i += nw) {
    const int64_t ob = old_ptr[i], on = old_ptr[i + 1] - ob;
    const int64_t ab = add_ptr[i], an = add_ptr[i + 1] - ab;
    const int64_t nb = new_ptr[i];
    if (an == 0) {
      for (int64_t j = lane; j < on; j += 32) new_col[nb + j] = old_col[ob + j];
      continue;
    }
    for (int64_t j = lane; j < on; j += 32) {
      const int32_t c = old_col[ob + j];
      new_col[nb + j + rank_lt(add_col + ab, an, c)] = c;
    }
    for (int64_t j = lane; j < an; j += 32) {
      const int32_t c = add_col[ab + j];
      new_col[nb + j + rank_lt(old_col + ob, on, c)] = c;   // c is not in the old row
    }
  }
}

__global__ void k_cols_of_keys(int64_t nnz, const unsigned long long* keys, int32_t* col) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    col[e] = (int32_t)(keys[e] & 0xffffffffull);
}

}  // namespace

void append_csr(CsrDevice& csr, int64_t m, const int64_t* d_src, const int64_t* d_dst,
                cudaStream_t st) {
  const int64_t n = csr.n;
  if (m <= 0) return;
  keep_pool();
  DevBuf<unsigned long long> counters(2, st);
  DevBuf<int> flags(2, st);
  OFSC_CUDA(cudaMemsetAsync(counters.p, 0, 2 * sizeof(unsigned long long), st));
  OFSC_CUDA(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), st));
  // 1. batch keys, sort, unique (within the batch)
  DevBuf<unsigned long long> ukeys(m, st);
  int64_t E = 0, loops = 0;
  {
    DevBuf<unsigned long long> keys(m, st), sorted(m, st);
    k_make_keys<<<blocks_for(m), 256, 0, st>>>(m, n, d_src, d_dst, keys.p, counters.p, flags.p);
    OFSC_LAUNCH_CHECK();
    size_t tb = 0;
    OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.p, sorted.p, m, 0, 64, st));
    {
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, sorted.p, m, 0, 64, st));
    }
    DevBuf<int64_t> nsel(1, st);
    tb = 0;
    OFSC_CUDA(cub::DeviceSelect::Unique(nullptr, tb, sorted.p, ukeys.p, nsel.p, m, st));
    {
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceSelect::Unique(tmp.p, tb, sorted.p, ukeys.p, nsel.p, m, st));
    }
    int64_t h_nsel = 0;
    unsigned long long h_cnt[2];
    int h_flags[2];
    OFSC_CUDA(cudaMemcpyAsync(&h_nsel, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(h_cnt, counters.p, sizeof(h_cnt), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(h_flags, flags.p, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaStreamSynchronize(st));
    OFSC_REQUIRE(!h_flags[0], OFSC_ERR_RANGE, "edge endpoint outside [0, n)");
    loops = (int64_t)h_cnt[0];
    unsigned long long last = 0;
    if (h_nsel > 0)
      OFSC_CUDA(cudaMemcpy(&last, ukeys.p + h_nsel - 1, sizeof(last), cudaMemcpyDeviceToHost));
    E = h_nsel - ((h_nsel > 0 && last == kSentinel) ? 1 : 0);
  }
  int64_t nadd = 0;
  DevBuf<unsigned long long> addk(E > 0 ? 2 * E : 1, st);
  if (E > 0) {
    // 2. symmetrise + sort by (row, col); 3. drop keys present in the old CSR
    DevBuf<unsigned long long> sym(2 * E, st), sym_sorted(2 * E, st);
    k_symmetrise<<<blocks_for(E), 256, 0, st>>>(E, ukeys.p, sym.p);
    OFSC_LAUNCH_CHECK();
    int hi = 1;
    while ((int64_t(1) << hi) < n) ++hi;
    size_t tb = 0;
    OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, sym.p, sym_sorted.p, 2 * E, 0, 32 + hi, st));
    {
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, sym.p, sym_sorted.p, 2 * E, 0, 32 + hi, st));
    }
    DevBuf<int> keep(2 * E, st);
    k_exists<<<blocks_for(2 * E), 256, 0, st>>>(2 * E, sym_sorted.p, csr.row_ptr, csr.col, keep.p);
    OFSC_LAUNCH_CHECK();
    DevBuf<int64_t> nsel(1, st);
    tb = 0;
    OFSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sym_sorted.p, keep.p, addk.p, nsel.p, 2 * E, st));
    {
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, sym_sorted.p, keep.p, addk.p, nsel.p, 2 * E,
                                           st));
    }
    OFSC_CUDA(cudaMemcpyAsync(&nadd, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t e_new = nadd / 2;                 // symmetric: both directions dropped together
  csr.n_loops += loops;
  csr.n_dups += m - loops - e_new;
  if (nadd == 0) return;
  // 4. degrees and row pointers
  DevBuf<int> deg_old(n, st), deg_add(n, st), deg(n, st);
  DevBuf<int64_t> deg64(n, st), add64(n, st), add_ptr(n + 1, st);
  OFSC_CUDA(cudaMemsetAsync(deg_add.p, 0, n * sizeof(int), st));
  k_old_degree<<<blocks_for(n), 256, 0, st>>>(n, csr.row_ptr, deg_old.p);
  k_add_degree<<<blocks_for(nadd), 256, 0, st>>>(nadd, addk.p, deg_add.p);
  OFSC_LAUNCH_CHECK();
  k_deg_to_i64<<<blocks_for(n), 256, 0, st>>>(n, deg_add.p, add64.p);
  k_sum_deg<<<blocks_for(n), 256, 0, st>>>(n, deg_old.p, deg_add.p, deg.p, deg64.p);
  OFSC_LAUNCH_CHECK();
  const int64_t nnz_new = csr.nnz + nadd;
  int64_t* new_ptr = nullptr;
  int32_t* new_col = nullptr;
  OFSC_CUDA(cudaMallocAsync(&new_ptr, (n + 1) * sizeof(int64_t), st));
  OFSC_CUDA(cudaMallocAsync(&new_col, nnz_new * sizeof(int32_t), st));
  {
    size_t tb = 0;
    OFSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg64.p, new_ptr, n, st));
    DevBuf<char> tmp(tb, st);
    OFSC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg64.p, new_ptr, n, st));
    OFSC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, add64.p, add_ptr.p, n, st));
  }
  OFSC_CUDA(cudaMemcpyAsync(add_ptr.p + n, &nadd, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  // 5. merge
  {
    DevBuf<int32_t> add_col(nadd, st);
    k_cols_of_keys<<<blocks_for(nadd), 256, 0, st>>>(nadd, addk.p, add_col.p);
    OFSC_LAUNCH_CHECK();
    const int64_t warps_blocks = (n * 32 + 255) / 256;
    const int nbm = (int)std::min<int64_t>(warps_blocks, (int64_t)num_sms() * 16);
    k_merge_rows<<<nbm, 256, 0, st>>>(n, csr.row_ptr, csr.col, add_ptr.p, add_col.p, new_ptr,
                                      new_col);
    OFSC_LAUNCH_CHECK();
    OFSC_CUDA(cudaStreamSynchronize(st));
  }
  dev_free(csr.row_ptr);   // stream synchronised above
  dev_free(csr.col);
  csr.row_ptr = new_ptr;
  csr.col = new_col;
  csr.nnz = nnz_new;
  csr.m_kept += e_new;
  // 6. s, isolated count, max degree, ||A||_F^2 (as in build_csr)
  k_scale<<<blocks_for(n), 256, 0, st>>>(n, deg.p, csr.s, csr.row_ptr + n, counters.p + 1,
                                         flags.p + 1, csr.nnz);
  OFSC_LAUNCH_CHECK();
  const int nb = blocks_for(n) < 1024 ? blocks_for(n) : 1024;
  DevBuf<double> part(nb, st);
  k_fro2<<<nb, 256, 0, st>>>(n, csr.row_ptr, csr.col, csr.s, part.p);
  OFSC_LAUNCH_CHECK();
  std::vector<double> hp(nb);
  unsigned long long iso = 0;
  int md = 0;
  OFSC_CUDA(cudaMemcpyAsync(hp.data(), part.p, nb * sizeof(double), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&iso, counters.p + 1, sizeof(iso), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&md, flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
  double f = 0.0;
  for (int b = 0; b < nb; ++b) f += hp[b];
  csr.fro2 = (double)n + f;
  csr.n_isolated = (int64_t)iso;
  csr.max_deg = md;
}

// ---- multi-GPU layout helpers ----------------------------------------------
__global__ void k_scatter_slots(const double* s, int64_t n, double* s_slot, float* s32_slot,
                                const int64_t* begins, int p, int64_t slot_rows) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    int r = 0;
    while (r + 1 < p && begins[r + 1] <= g) ++r;
    const int64_t id = r * slot_rows + (g - begins[r]);
    s_slot[id] = s[g];
    s32_slot[id] = (float)s[g];
  }
}

void scatter_slots(const double* s, int64_t n, double* s_slot, float* s32_slot,
                   const int64_t* d_begins, int p, int64_t slot_rows, cudaStream_t st) {
  k_scatter_slots<<<blocks_for(n), 256, 0, st>>>(s, n, s_slot, s32_slot, d_begins, p, slot_rows);
  OFSC_LAUNCH_CHECK();
}

// ---- halo layout (p > 1) -----------------------------
// A rank's gather buffer holds its own rows (ext ids 0..n_local-1) followed by
// the remote rows its columns reference ("halo"), in ascending global id, so
// the rows owned by peer q form one contiguous segment.  The graph is
// symmetric, so the rows q must send to r -- q's rows with a neighbour in r's
// range -- are exactly r's halo segment from q, in the same (ascending) order:
// both sides derive the exchange plan from the CSR alone, with no handshake.
namespace {

__device__ __forceinline__ int owner_of(int64_t g, const int64_t* begins, int p) {
  int r = 0;
  while (r + 1 < p && begins[r + 1] <= g) ++r;
  return r;
}

__global__ void k_remote_flags(int64_t nnz, const int32_t* col, int64_t rb, int64_t re, int* flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (col[e] < rb || col[e] >= re) ? 1 : 0;
}

__global__ void k_remap_ext(int64_t nnz, const int32_t* col, int64_t rb, int64_t re,
                            int64_t n_local, const int32_t* halo, int64_t h, int32_t* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = col[e];
    if (c >= rb && c < re) {
      out[e] = (int32_t)(c - rb);
    } else {
      int64_t lo = 0, hi = h;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (halo[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      out[e] = (int32_t)(n_local + lo);
    }
  }
}

// flag[r * n_local + i] = 1 iff own row i has a neighbour owned by rank r != self
__global__ void k_send_flags(int64_t n_local, const int64_t* row_ptr, const int32_t* col,
                             const int64_t* begins, int p, int self, unsigned char* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < n_local; i += nw)
    for (int64_t q = row_ptr[i] + lane; q < row_ptr[i + 1]; q += 32) {
      const int r = owner_of(col[q], begins, p);
      if (r != self) flag[(int64_t)r * n_local + i] = 1;   // benign race: all write 1
    }
}

__global__ void k_gather_s(int64_t rows, const int32_t* gid, const double* s, double* s_ext,
                           float* s32_ext) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = gid[e] >= 0 ? s[gid[e]] : 0.0;
    s_ext[e] = v;
    s32_ext[e] = (float)v;
  }
}

__global__ void k_local_count(int64_t n_local, const int64_t* row_ptr, const int32_t* col,
                              int64_t* cnt_loc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_local;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) c += col[q] < n_local;
    cnt_loc[i] = c;
  }
}

// stable split of every row's columns: local ext ids (< n_local) | halo ext ids
__global__ void k_split_rows(int64_t n_local, const int64_t* row_ptr, const int32_t* col,
                             const int64_t* ptr_loc, int32_t* col_loc, int32_t* col_rem) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_local;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = ptr_loc[i], b = row_ptr[i] - ptr_loc[i];   // remote offset = row_ptr - ptr_loc
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      const int32_t c = col[q];
      if (c < n_local) col_loc[a++] = c;
      else col_rem[b++] = c;
    }
  }
}

__global__ void k_sub_ptr(int64_t n1, const int64_t* a, const int64_t* b, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

__global__ void k_iota32(int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

}  // namespace

void build_halo(const CsrDevice& csr, const int64_t* h_begins, const int64_t* d_begins, int p,
                int rank, HaloLayout& out, cudaStream_t st) {
  keep_pool();
  const int64_t rb = h_begins[rank], re = h_begins[rank + 1];
  const int64_t nl = re - rb;
  std::vector<int64_t> rp_ends(2);
  OFSC_CUDA(cudaMemcpyAsync(&rp_ends[0], csr.row_ptr + rb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&rp_ends[1], csr.row_ptr + re, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
  const int64_t e0 = rp_ends[0], nnz = rp_ends[1] - rp_ends[0];
  const int32_t* gcol = csr.col + e0;
  out.n_local = nl;
  // 1. halo ids: unique remote columns, ascending
  int64_t h = 0;
  DevBuf<int32_t> halo(nnz > 0 ? nnz : 1, st);
  if (nnz > 0) {
    DevBuf<int> flag(nnz, st);
    DevBuf<int32_t> rem(nnz, st), rem_sorted(nnz, st);
    DevBuf<int64_t> nsel(1, st);
    k_remote_flags<<<blocks_for(nnz), 256, 0, st>>>(nnz, gcol, rb, re, flag.p);
    OFSC_LAUNCH_CHECK();
    size_t tb = 0;
    OFSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, gcol, flag.p, rem.p, nsel.p, nnz, st));
    {
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, gcol, flag.p, rem.p, nsel.p, nnz, st));
    }
    int64_t nrem = 0;
    OFSC_CUDA(cudaMemcpyAsync(&nrem, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaStreamSynchronize(st));
    if (nrem > 0) {
      tb = 0;
      OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, rem.p, rem_sorted.p, nrem, 0, 32, st));
      {
        DevBuf<char> tmp(tb, st);
        OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, rem.p, rem_sorted.p, nrem, 0, 32, st));
      }
      tb = 0;
      OFSC_CUDA(cub::DeviceSelect::Unique(nullptr, tb, rem_sorted.p, halo.p, nsel.p, nrem, st));
      {
        DevBuf<char> tmp(tb, st);
        OFSC_CUDA(cub::DeviceSelect::Unique(tmp.p, tb, rem_sorted.p, halo.p, nsel.p, nrem, st));
      }
      OFSC_CUDA(cudaMemcpyAsync(&h, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      OFSC_CUDA(cudaStreamSynchronize(st));
    }
  }
  out.ext_rows = nl + h;
  out.h_gid.resize(out.ext_rows);
  for (int64_t i = 0; i < nl; ++i) out.h_gid[i] = (int32_t)(rb + i);
  if (h > 0)
    OFSC_CUDA(cudaMemcpy(out.h_gid.data() + nl, halo.p, h * sizeof(int32_t), cudaMemcpyDeviceToHost));
  dev_alloc((void**)&out.d_gid, std::max<int64_t>(out.ext_rows, 1) * sizeof(int32_t), st);
  OFSC_CUDA(cudaMemcpy(out.d_gid, out.h_gid.data(), out.ext_rows * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  // 2. local CSR: rebased row pointers, columns -> ext ids; s on the ext rows
  dev_alloc((void**)&out.row_ptr, (nl + 1) * sizeof(int64_t), st);
  dev_alloc((void**)&out.col, std::max<int64_t>(nnz, 1) * sizeof(int32_t), st);
  rebase_row_ptr(csr.row_ptr + rb, nl, e0, out.row_ptr, st);
  if (nnz > 0) {
    k_remap_ext<<<blocks_for(nnz), 256, 0, st>>>(nnz, gcol, rb, re, nl, halo.p, h, out.col);
    OFSC_LAUNCH_CHECK();
  }
  out.nnz_local = nnz;
  // 2b. the same CSR split per row into local columns | halo columns (order kept):
  //     the local part runs while the halo is exchanged
  {
    DevBuf<int64_t> cnt(std::max<int64_t>(nl, 1), st);
    dev_alloc((void**)&out.row_ptr_loc, (nl + 1) * sizeof(int64_t), st);
    dev_alloc((void**)&out.row_ptr_rem, (nl + 1) * sizeof(int64_t), st);
    dev_alloc((void**)&out.col_loc, std::max<int64_t>(nnz, 1) * sizeof(int32_t), st);
    dev_alloc((void**)&out.col_rem, std::max<int64_t>(nnz, 1) * sizeof(int32_t), st);
    OFSC_CUDA(cudaMemsetAsync(out.row_ptr_loc, 0, (nl + 1) * sizeof(int64_t), st));
    if (nl > 0) {
      k_local_count<<<blocks_for(nl), 256, 0, st>>>(nl, out.row_ptr, out.col, cnt.p);
      OFSC_LAUNCH_CHECK();
      size_t tb = 0;
      OFSC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.p, out.row_ptr_loc + 1, nl, st));
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, cnt.p, out.row_ptr_loc + 1, nl, st));
      k_sub_ptr<<<blocks_for(nl + 1), 256, 0, st>>>(nl + 1, out.row_ptr, out.row_ptr_loc,
                                                     out.row_ptr_rem);
      k_split_rows<<<blocks_for(nl), 256, 0, st>>>(nl, out.row_ptr, out.col, out.row_ptr_loc,
                                                  out.col_loc, out.col_rem);
      OFSC_LAUNCH_CHECK();
    } else {
      OFSC_CUDA(cudaMemsetAsync(out.row_ptr_rem, 0, sizeof(int64_t), st));
    }
  }
  dev_alloc((void**)&out.s_ext, std::max<int64_t>(out.ext_rows, 1) * sizeof(double), st);
  dev_alloc((void**)&out.s32_ext, std::max<int64_t>(out.ext_rows, 1) * sizeof(float), st);
  k_gather_s<<<blocks_for(std::max<int64_t>(out.ext_rows, 1)), 256, 0, st>>>(
      out.ext_rows, out.d_gid, csr.s, out.s_ext, out.s32_ext);
  OFSC_LAUNCH_CHECK();
  // 3. receive plan: halo segment owned by each peer
  out.recv_cnt.assign(p, 0);
  out.recv_off.assign(p, nl);
  for (int q = 0; q < p; ++q) {
    const auto lo = std::lower_bound(out.h_gid.begin() + nl, out.h_gid.end(), (int32_t)h_begins[q]);
    const auto hi = std::lower_bound(out.h_gid.begin() + nl, out.h_gid.end(), (int32_t)h_begins[q + 1]);
    out.recv_off[q] = lo - out.h_gid.begin();
    out.recv_cnt[q] = hi - lo;
  }
  // 4. send plan: own rows with a neighbour owned by each peer (ascending)
  out.send_cnt.assign(p, 0);
  out.send_off.assign(p + 1, 0);
  DevBuf<unsigned char> sflag((size_t)p * std::max<int64_t>(nl, 1), st);
  OFSC_CUDA(cudaMemsetAsync(sflag.p, 0, (size_t)p * std::max<int64_t>(nl, 1), st));
  if (nnz > 0) {
    const int64_t wb = (nl * 32 + 255) / 256;
    k_send_flags<<<(int)std::min<int64_t>(std::max<int64_t>(wb, 1), (int64_t)num_sms() * 16), 256, 0,
                   st>>>(nl, csr.row_ptr + rb, csr.col, d_begins, p, rank, sflag.p);
    // (global row pointers: absolute offsets into the full csr.col)
    OFSC_LAUNCH_CHECK();
  }
  std::vector<int32_t> send_idx;
  {
    DevBuf<int32_t> iota(std::max<int64_t>(nl, 1), st), sel(std::max<int64_t>(nl, 1), st);
    DevBuf<int64_t> nsel(1, st);
    k_iota32<<<blocks_for(std::max<int64_t>(nl, 1)), 256, 0, st>>>(nl, iota.p);
    OFSC_LAUNCH_CHECK();
    for (int q = 0; q < p; ++q) {
      out.send_off[q + 1] = out.send_off[q];
      if (q == rank || nl == 0) continue;
      size_t tb = 0;
      OFSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, sflag.p + (size_t)q * nl, sel.p,
                                           nsel.p, nl, st));
      DevBuf<char> tmp(tb, st);
      OFSC_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, iota.p, sflag.p + (size_t)q * nl, sel.p,
                                           nsel.p, nl, st));
      int64_t cnt = 0;
      OFSC_CUDA(cudaMemcpyAsync(&cnt, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      OFSC_CUDA(cudaStreamSynchronize(st));
      const size_t old = send_idx.size();
      send_idx.resize(old + cnt);
      if (cnt > 0)
        OFSC_CUDA(cudaMemcpy(send_idx.data() + old, sel.p, cnt * sizeof(int32_t),
                             cudaMemcpyDeviceToHost));
      out.send_cnt[q] = cnt;
      out.send_off[q + 1] = out.send_off[q] + cnt;
    }
  }
  out.total_send = (int64_t)send_idx.size();
  dev_alloc((void**)&out.d_send_idx, std::max<int64_t>(out.total_send, 1) * sizeof(int32_t), st);
  if (out.total_send > 0)
    OFSC_CUDA(cudaMemcpy(out.d_send_idx, send_idx.data(), out.total_send * sizeof(int32_t),
                         cudaMemcpyHostToDevice));
  OFSC_CUDA(cudaStreamSynchronize(st));
}

__global__ void k_rebase(const int64_t* in, int64_t rows, int64_t base, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= rows;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] - base;
}

void rebase_row_ptr(const int64_t* in, int64_t rows, int64_t base, int64_t* out, cudaStream_t st) {
  k_rebase<<<blocks_for(rows + 1), 256, 0, st>>>(in, rows, base, out);
  OFSC_LAUNCH_CHECK();
}

// ---- locality reordering: label propagation (graph-derived communities) ----
// Semi-synchronous LPA: each sweep updates the nodes of one hash colour, then
// the other, from a double-buffered label array (a pure function of the input
// labels: deterministic).  A node takes the most frequent label among its first
// kLpaCap neighbours; ties go to the smallest hash(label, sweep); it keeps its
// own label if that ties the maximum.  Nodes are then ordered by (label, id) so
// that communities occupy contiguous row ranges and the SpMM's neighbour
// gathers stay in L2.
constexpr int kLpaCap = 128;
constexpr int kLpaSlots = 256;

__device__ __forceinline__ uint32_t mix32(uint32_t x, uint32_t seed) {
  uint64_t z = (uint64_t)x * 0x9E3779B97F4A7C15ull + (uint64_t)seed * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 31;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 29;
  return (uint32_t)z;
}

__global__ void __launch_bounds__(256) k_lpa_pass(int64_t n, const int64_t* __restrict__ row_ptr,
                                                  const int32_t* __restrict__ col,
                                                  const int* __restrict__ lin, int* __restrict__ lout,
                                                  int colour, uint32_t seed,
                                                  unsigned long long* changes, int fast) {
  __shared__ int keys[8][kLpaSlots];
  __shared__ int cnts[8][kLpaSlots];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int* K = keys[w];
  int* Cn = cnts[w];
  unsigned long long nchg = 0;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t i = (int64_t)blockIdx.x * 8 + w; i < n; i += nw) {
    const int own = lin[i];
    if ((int)(mix32((uint32_t)i, 0x5EEDu) & 1u) != colour) {
      if (lane == 0) lout[i] = own;
      continue;
    }
    const int64_t beg = row_ptr[i];
    const int deg = (int)min((int64_t)kLpaCap, row_ptr[i + 1] - beg);
    if (deg == 0) {
      if (lane == 0) lout[i] = own;
      continue;
    }
    if (deg <= 32 && fast) {
      // one neighbour per lane: __match_any_sync groups the lanes holding the same
      // label, so its popcount is that label's count (no table, no atomics); the
      // selection below is the table path's (count, hash, label) rule exactly
      const bool has = lane < deg;
      const int L = has ? lin[col[beg + lane]] : -1 - lane;   // padding lanes: singletons
      const unsigned m = __match_any_sync(0xffffffffu, L);
      const int c = has ? __popc(m) : 0;
      int owncnt = (has && L == own) ? c : 0;
      int bc = has ? c : 0, bl = has ? L : -1;
      uint32_t bh = has ? mix32((uint32_t)L, seed) : 0xffffffffu;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const uint32_t oh = __shfl_xor_sync(0xffffffffu, bh, o);
        if (oc > bc || (oc == bc && (oh < bh || (oh == bh && ol < bl)))) {
          bc = oc;
          bl = ol;
          bh = oh;
        }
        owncnt = max(owncnt, __shfl_xor_sync(0xffffffffu, owncnt, o));
      }
      const int nl = (owncnt >= bc) ? own : bl;
      if (lane == 0) {
        lout[i] = nl;
        nchg += nl != own;
      }
      continue;
    }
    // open-addressing table sized to the (capped) degree: >= 2 deg slots, >= 32
    int S = 32;
    while (S < 2 * deg) S <<= 1;
    const int mask = S - 1;
    for (int q = lane; q < S; q += 32) {
      K[q] = -1;
      Cn[q] = 0;
    }
    __syncwarp();
    for (int e = lane; e < deg; e += 32) {
      const int L = lin[col[beg + e]];
      int slot = (int)(mix32((uint32_t)L, 7u) & (uint32_t)mask);
      while (true) {
        const int prev = atomicCAS(&K[slot], -1, L);
        if (prev == -1 || prev == L) {
          atomicAdd(&Cn[slot], 1);
          break;
        }
        slot = (slot + 1) & mask;
      }
    }
    __syncwarp();
    int bc = 0, bl = -1, owncnt = 0;
    uint32_t bh = 0xffffffffu;
    for (int q = lane; q < S; q += 32) {
      const int L = K[q];
      if (L < 0) continue;
      const int c = Cn[q];
      if (L == own) owncnt = c;
      const uint32_t h = mix32((uint32_t)L, seed);
      if (c > bc || (c == bc && (h < bh || (h == bh && L < bl)))) {
        bc = c;
        bl = L;
        bh = h;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      const uint32_t oh = __shfl_xor_sync(0xffffffffu, bh, o);
      if (oc > bc || (oc == bc && (oh < bh || (oh == bh && ol < bl)))) {
        bc = oc;
        bl = ol;
        bh = oh;
      }
      owncnt = max(owncnt, __shfl_xor_sync(0xffffffffu, owncnt, o));
    }
    const int nl = (owncnt >= bc) ? own : bl;
    if (lane == 0) {
      lout[i] = nl;
      nchg += nl != own;
    }
    __syncwarp();
  }
  if (lane == 0 && nchg) atomicAdd(changes, nchg);
}

__global__ void k_lpa_keys(int64_t n, const int* lab, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((unsigned long long)(unsigned)lab[i] << 32) | (unsigned long long)i;
}

__global__ void k_perm_from_keys(int64_t n, const unsigned long long* keys, int32_t* perm,
                                 int32_t* inv, int* flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t node = (int32_t)(keys[j] & 0xffffffffull);
    perm[j] = node;
    inv[node] = (int32_t)j;
    flag[j] = (j == 0 || (keys[j] >> 32) != (keys[j - 1] >> 32)) ? 1 : 0;
  }
}

// cid[j] = community index of internal row j (scan of the start flags); cstart[c] = first row
__global__ void k_comm_index(int64_t n, const int* flag, const int* scan, int32_t* cid,
                             int64_t* cstart) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int c = scan[j] - 1;
    cid[j] = c;
    if (flag[j]) cstart[c] = j;
  }
}

__global__ void k_intra_edges(int64_t n, const int64_t* row_ptr, const int32_t* col, const int* lab,
                              unsigned long long* cnt) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) c += lab[col[q]] == lab[i];
  if (c) atomicAdd(cnt, c);
}

// endpoints outside [0, n) are not looked up: they become -1, which the CSR build /
// merge that follows rejects with OFSC_ERR_RANGE (k_make_keys)
__global__ void k_relabel_edges(int64_t m, int64_t n, const int64_t* src, const int64_t* dst,
                                const int32_t* inv, int64_t* s2, int64_t* d2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = src[e], v = dst[e];
    s2[e] = (u >= 0 && u < n) ? (int64_t)inv[u] : -1;
    d2[e] = (v >= 0 && v < n) ? (int64_t)inv[v] : -1;
  }
}

__global__ void k_iota(int64_t n, int* lab) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lab[i] = (int)i;
}

void lpa_order(const CsrDevice& csr, int sweeps, int32_t* d_perm, int32_t* d_inv, int64_t* n_comm,
               double* intra_frac, int32_t* d_cid, int64_t** d_cstart, cudaStream_t st) {
  const int64_t n = csr.n;
  DevBuf<int> la(n, st), lb(n, st), cnt(1, st);
  DevBuf<unsigned long long> keys(n, st), sorted(n, st), ic(1, st);
  k_iota<<<blocks_for(n), 256, 0, st>>>(n, la.p);
  OFSC_LAUNCH_CHECK();
  int* cur = la.p;
  int* nxt = lb.p;
  const int nb = num_sms() * 8;
  static const int fast = [] {          // OFSC_LPA_FAST=0: table path for every node (A/B)
    const char* e = getenv("OFSC_LPA_FAST");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  // sweeps until fewer than n/1000 labels change (at least 6, at most `sweeps`)
  unsigned long long chg = 0, *h_chg = &chg;   // pageable: no pinned alloc / free (device syncs)
  for (int sw = 0; sw < sweeps; ++sw) {
    OFSC_CUDA(cudaMemsetAsync(ic.p, 0, sizeof(unsigned long long), st));
    for (int colour = 0; colour < 2; ++colour) {
      k_lpa_pass<<<nb, 256, 0, st>>>(n, csr.row_ptr, csr.col, cur, nxt, colour,
                                     (uint32_t)(2 * sw + colour + 1), ic.p, fast);
      OFSC_LAUNCH_CHECK();
      std::swap(cur, nxt);
    }
    if (sw >= 5) {
      OFSC_CUDA(cudaMemcpyAsync(h_chg, ic.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      OFSC_CUDA(cudaStreamSynchronize(st));
      if (*h_chg * 1000ull < (unsigned long long)n) break;
    }
  }
  k_lpa_keys<<<blocks_for(n), 256, 0, st>>>(n, cur, keys.p);
  OFSC_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  OFSC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, n, 0, 64, st));
  {
    DevBuf<char> tmp(tmp_bytes, st);
    OFSC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, n, 0, 64, st));
  }
  OFSC_CUDA(cudaMemsetAsync(ic.p, 0, sizeof(unsigned long long), st));
  DevBuf<int> flag(n, st), scan(n, st);
  k_perm_from_keys<<<blocks_for(n), 256, 0, st>>>(n, sorted.p, d_perm, d_inv, flag.p);
  OFSC_LAUNCH_CHECK();
  {
    size_t tb = 0;
    OFSC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, flag.p, scan.p, n, st));
    DevBuf<char> tmp(tb, st);
    OFSC_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, flag.p, scan.p, n, st));
  }
  OFSC_CUDA(cudaMemcpyAsync(cnt.p, scan.p + n - 1, sizeof(int), cudaMemcpyDeviceToDevice, st));
  k_intra_edges<<<blocks_for(n), 256, 0, st>>>(n, csr.row_ptr, csr.col, cur, ic.p);
  OFSC_LAUNCH_CHECK();
  int h_cnt = 0;
  unsigned long long h_ic = 0;
  OFSC_CUDA(cudaMemcpyAsync(&h_cnt, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaMemcpyAsync(&h_ic, ic.p, sizeof(h_ic), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
  *n_comm = h_cnt;
  *intra_frac = csr.nnz > 0 ? (double)h_ic / (double)csr.nnz : 1.0;
  dev_alloc((void**)d_cstart, (h_cnt + 1) * sizeof(int64_t), st);
  k_comm_index<<<blocks_for(n), 256, 0, st>>>(n, flag.p, scan.p, d_cid, *d_cstart);
  OFSC_LAUNCH_CHECK();
  OFSC_CUDA(cudaMemcpyAsync(*d_cstart + h_cnt, &n, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
}

void relabel_edges(int64_t m, int64_t n, const int64_t* src, const int64_t* dst,
                   const int32_t* inv, int64_t* s2, int64_t* d2, cudaStream_t st) {
  if (m <= 0) return;
  k_relabel_edges<<<blocks_for(m), 256, 0, st>>>(m, n, src, dst, inv, s2, d2);
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

// C2a: the SpMM of the SpMM + Gram step (eq:spmm P:440,
// P:468-487).
//
//   Y_i = (A Z)_i = -Z_i - s_i * sum_{j in N(i)} s_j Z_j        (A = L - 2I)
//
// A group of KP/4 lanes owns a row and gathers its neighbour rows of Z with
// 16-byte vector loads (each load instruction covers a contiguous half row),
// 8 neighbour rows in flight per group, summing in CSR (ascending column)
// order; rows are handed out in order from a global counter so the gathered
// window stays L2-resident on locality-ordered graphs.  The Grams of the step
// are NOT formed here: they are computed by the TMA-streamed DMMA kernel C2b
// (k_gram_stream_ws, kernels_stream.cu) right after, over the SpMM's output
// (launch_spmm_then_gram).  A fused SpMM + Gram kernel was measured worse on
// B200: the gathers need all 24 warps and the L1 of the SM as landing space
// (c4 SpMM 5.20 ms at 3 CTAs/SM, 6.95 ms at 2, 12.8 ms at 1:
// tools/spmm_occupancy.py, profiles/r02), so there are no registers or
// shared memory left for DMMA accumulators without slowing the gathers by
// more than C2b costs.
//   mode 0 (iteration):  C2b T = Z^T Y, R' = X^T Y    (Z = V)
//   mode 1 (refresh):    C2b M = Z^T Z, W = Z^T Y     (Z = X)
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "sm100.cuh"

namespace ofsc {

// C2a: Y = A Z on the column window [c0, c0 + CW) (CW = KP: one pass; CW < KP:
// KP/CW passes, each gathering CW-column row segments, so the gathered working
// set of a community is CW/KP of its rows' bytes and stays L2-resident).
// A group of LPR = CW/4 lanes owns a row (each lane 4 consecutive columns = two
// 16-byte loads per neighbour), RPW = 32/LPR rows per warp; no shared memory and
// no barriers, so warps stream independently and the register file holds only
// accumulators and in-flight neighbour rows (8 per row).
// L2 eviction-priority hints (HINT = 1, reordered graphs): the column ids,
// the output rows and neighbour rows outside the row's community are loaded /
// stored evict_first, so the current community's rows (reused ~15 times while
// its rows are processed) keep the L2.
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ldg2h(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ldg2h(const float* p, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldg1h(const int32_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg2h(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol));
}
__device__ __forceinline__ void stg2h(float* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y),
               "l"(pol));
}

// SV = 2: the column stream holds (column id | degree of the column's node << 23)
// and s_j is read from a per-degree table (sval = table[max_deg + 1]), so one 4-byte
// stream replaces the column ids AND the 8-byte per-nonzero s_j stream
constexpr int kPackShift = 23;
constexpr int kPackMask = (1 << kPackShift) - 1;
template <int SV>
__device__ __forceinline__ int col_id(int raw) {
  if constexpr (SV == 2) return raw & kPackMask;
  else return raw;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <typename T, int KP, int CW, int HINT, int PHASE, int SV = 0, int PF = 0, int NIF = 8>
__global__ void __launch_bounds__(kThreads, NIF >= 8 ? 3 : (NIF >= 6 ? 4 : 5))
k_spmm(int64_t n_local, int64_t own_off, const int64_t* __restrict__ row_ptr,
       const int32_t* __restrict__ col, const double* __restrict__ s,
       const float* __restrict__ s32, const T* __restrict__ Zg, T* __restrict__ Y,
       const int* stop, unsigned long long* __restrict__ ctr, int ch, int c0,
       const int32_t* __restrict__ cid, const int64_t* __restrict__ cstart, int64_t heavy,
       const T* __restrict__ sval) {
  // SV = 1: the neighbour scale s_j is read from the per-nonzero array sval (streamed
  // with the column ids) instead of gathered from s by column id
  // rows with more than `heavy` neighbours are left to the chunked heavy-row pass
  // PHASE 0: Y = A Z (whole rows); 1: Y <- raw neighbour sums over this CSR (the
  // local columns of a multi-GPU rank, while the halo is in flight); 2: continue
  // the sums from Y over this CSR (the halo columns) and finish Y = -Z_i - s_i sum
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  uint64_t pf = 0, pn = 0;
  if constexpr (HINT) {
    pf = pol_evict_first();
    pn = pol_evict_normal();
  }
  using V2 = typename Vec2<T>::type;
  constexpr int LPR = CW / 4;
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, l = lane % LPR;
  const bool active = sub < RPW;                // KP = 48: lanes 24..31 idle
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // lane l of a row group owns columns {2l, 2l+1} and {CW/2 + 2l, CW/2 + 2l + 1}:
  // each of the two 16-byte loads of a neighbour row then covers a contiguous
  // half of the row segment (whole 32-byte sectors, no L1 re-reads)
  constexpr int H2 = CW / 2;
  const T* zc = Zg + c0 + 2 * l;
  // Rows are handed out in order in chunks of kSpmmChunk from a global counter
  // (ctr != NULL), so all warps work on a narrow, advancing window of rows and
  // the neighbour rows of the current (reordered) community stay in L2;
  // ctr == NULL: static interleaved assignment.
  const int CH = ch;
  int64_t round = 0;
  auto grab = [&]() -> int64_t {
    if (ctr) {
      unsigned long long b0 = 0;
      if (lane == 0) b0 = atomicAdd(ctr, (unsigned long long)CH);
      return (int64_t)__shfl_sync(0xffffffffu, b0, 0);
    }
    const int64_t b = (gw + round * nw) * CH;
    ++round;
    return b;
  };
  // PF >= 3: the next chunk is grabbed one chunk early, so the rows a group will sum
  // next (the next row pair of this chunk, or the first rows of the next chunk) can
  // have their first LPR neighbour rows prefetched into L2 while this row is summed
  int64_t base_next = grab();
  while (true) {
    const int64_t base = base_next;
    if (base >= n_local) break;
    if constexpr (PF >= 3) base_next = grab();
#pragma unroll 1
    for (int q = 0; q < CH; q += RPW) {
    const int64_t i = base + q + sub;
    if constexpr (PF >= 3) {
      const int64_t inext = (q + RPW < CH) ? i + RPW : base_next + sub;
      if (active && inext < n_local) {
        const int64_t nb = row_ptr[inext], ne = row_ptr[inext + 1];
        if (nb + l < ne && ne - nb <= heavy) {
          const char* rp = (const char*)(Zg + (int64_t)col_id<SV>(__ldg(col + nb + l)) * KP + c0);
#pragma unroll
          for (int b = 0; b < (int)(CW * sizeof(T)); b += 128) prefetch_l2(rp + b);
        }
      }
    }
    if (!active || i >= n_local) continue;
    const int64_t beg = row_ptr[i], end = row_ptr[i + 1];
    if (end - beg > heavy) continue;               // uniform within the row group
    int lo = 0, hi = 0;                            // community row range of row i (HINT)
    if constexpr (HINT) {
      const int ci = cid[i];
      lo = (int)cstart[ci];
      hi = (int)cstart[ci + 1];
    }
    T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if constexpr (PHASE == 2) {
      const T* yp = Y + i * KP + c0 + 2 * l;
      const V2 p0 = *reinterpret_cast<const V2*>(yp), p1 = *reinterpret_cast<const V2*>(yp + H2);
      a0 = p0.x;
      a1 = p0.y;
      a2 = p1.x;
      a3 = p1.y;
    }
    int64_t e = beg;
    if constexpr (PF >= 2) {
      // lane l prefetches (into L2) the whole row of neighbour beg + NIF + l: with the
      // NIF rows the registers hold, up to NIF + LPR neighbour rows of this row are in flight
      const int64_t qn = beg + NIF + l;
      if (qn < end) {
        const char* rp = (const char*)(Zg + (int64_t)col_id<SV>(__ldg(col + qn)) * KP + c0);
#pragma unroll
        for (int b = 0; b < (int)(CW * sizeof(T)); b += 128) prefetch_l2(rp + b);
      }
    }
    for (; e + NIF <= end; e += NIF) {
      int c[NIF];
      int dg[SV == 2 ? NIF : 1];
#pragma unroll
      for (int u = 0; u < NIF; ++u) {
        if constexpr (HINT) c[u] = ldg1h(col + e + u, pf);
        else c[u] = __ldg(col + e + u);
        if constexpr (SV == 2) {
          dg[u] = (int)((unsigned)c[u] >> kPackShift);
          c[u] &= kPackMask;
        }
      }
      if constexpr (PF >= 2) {
        // PF >= 2: lanes 0..NIF-1 of the group prefetch the whole rows of neighbours
        // e + 2 NIF .. e + 3 NIF - 1 (the row start covered e + NIF .. e + NIF + LPR - 1)
        const int64_t qn = e + 2 * NIF + l;
        if (e >= NIF && l < NIF && qn < end) {
          const char* rp = (const char*)(Zg + (int64_t)col_id<SV>(__ldg(col + qn)) * KP + c0);
#pragma unroll
          for (int b = 0; b < (int)(CW * sizeof(T)); b += 128) prefetch_l2(rp + b);
        }
      }
      if constexpr (PF == 1) {
        // PF = 1: the next batch's neighbour rows are prefetched into L2 (no register
        // destination), so twice as many rows are in flight as registers hold
        if (e + 2 * NIF <= end) {
#pragma unroll
          for (int u = 0; u < NIF; ++u) {
            const int cn = col_id<SV>(__ldg(col + e + NIF + u));
            prefetch_l2(zc + (int64_t)cn * KP);
            prefetch_l2(zc + (int64_t)cn * KP + H2);
          }
        }
      }
      V2 z0[NIF], z1[NIF];
      T sv[NIF];
#pragma unroll
      for (int u = 0; u < NIF; ++u) {
        if constexpr (HINT) {
          const T* zr = zc + (int64_t)c[u] * KP;
          const uint64_t pol = (c[u] >= lo && c[u] < hi) ? pn : pf;
          z0[u] = ldg2h(zr, pol);
          z1[u] = ldg2h(zr + H2, pol);
        } else {
          const T* zr = zc + (int64_t)c[u] * KP;
          z0[u] = __ldg(reinterpret_cast<const V2*>(zr));
          z1[u] = __ldg(reinterpret_cast<const V2*>(zr + H2));
        }
        if constexpr (SV == 2) sv[u] = __ldg(sval + dg[u]);
        else if constexpr (SV) sv[u] = __ldg(sval + e + u);
        else if constexpr (sizeof(T) == 8) sv[u] = (T)__ldg(s + c[u]);
        else sv[u] = (T)__ldg(s32 + c[u]);
      }
#pragma unroll
      for (int u = 0; u < NIF; ++u) {
        a0 = fma(sv[u], z0[u].x, a0);
        a1 = fma(sv[u], z0[u].y, a1);
        a2 = fma(sv[u], z1[u].x, a2);
        a3 = fma(sv[u], z1[u].y, a3);
      }
    }
    for (; e < end; ++e) {
      const int raw = __ldg(col + e);
      const int c = col_id<SV>(raw);
      const T* zr = zc + (int64_t)c * KP;
      const V2 z0 = __ldg(reinterpret_cast<const V2*>(zr));
      const V2 z1 = __ldg(reinterpret_cast<const V2*>(zr + H2));
      T sv;
      if constexpr (SV == 2) sv = __ldg(sval + ((unsigned)raw >> kPackShift));
      else if constexpr (SV) sv = __ldg(sval + e);
      else if constexpr (sizeof(T) == 8) sv = (T)__ldg(s + c);
      else sv = (T)__ldg(s32 + c);
      a0 = fma(sv, z0.x, a0);
      a1 = fma(sv, z0.y, a1);
      a2 = fma(sv, z1.x, a2);
      a3 = fma(sv, z1.y, a3);
    }
    V2 y0, y1;
    if constexpr (PHASE == 1) {                    // raw partial sums
      y0.x = a0;
      y0.y = a1;
      y1.x = a2;
      y1.y = a3;
    } else {
      const T* zo = Zg + (own_off + i) * KP + c0 + 2 * l;
      const V2 o0 = *reinterpret_cast<const V2*>(zo), o1 = *reinterpret_cast<const V2*>(zo + H2);
      T si;
      if constexpr (sizeof(T) == 8) si = (T)s[own_off + i];
      else si = s32[own_off + i];
      y0.x = -o0.x - si * a0;
      y0.y = -o0.y - si * a1;
      y1.x = -o1.x - si * a2;
      y1.y = -o1.y - si * a3;
    }
    if constexpr (HINT) {
      stg2h(Y + i * KP + c0 + 2 * l, y0, pf);
      stg2h(Y + i * KP + c0 + 2 * l + H2, y1, pf);
    } else {
      *reinterpret_cast<V2*>(Y + i * KP + c0 + 2 * l) = y0;
      *reinterpret_cast<V2*>(Y + i * KP + c0 + 2 * l + H2) = y1;
    }
    }
    if constexpr (PF < 3) base_next = grab();
  }
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// ---- degree-aware row binning (power-law rows) ------------------------------
// Chunk pass: one LPR-lane group per chunk of <= kHeavyChunk neighbours of a
// heavy row (same lane mapping and 8-in-flight loop as k_spmm); raw partial
// sums go to scratch[chunk].  Finalize: per (heavy row, column), the chunk
// partials summed in chunk order (deterministic), then the row finished as in
// k_spmm (PHASE 1 stores the raw sum, PHASE 2 adds the stored partial first).
template <typename T, int KP>
__global__ void __launch_bounds__(kThreads)
k_spmm_chunks(int64_t n_chunks, const int64_t* __restrict__ cbeg, const int64_t* __restrict__ cend,
              const int32_t* __restrict__ col, const double* __restrict__ s,
              const float* __restrict__ s32, const T* __restrict__ Zg, T* __restrict__ scratch,
              const int* stop) {
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  using V2 = typename Vec2<T>::type;
  constexpr int LPR = KP / 4;
  constexpr int RPW = 32 / LPR;
  constexpr int H2 = KP / 2;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, l = lane % LPR;
  if (sub >= RPW) return;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T* zc = Zg + 2 * l;
  for (int64_t q = gw * RPW + sub; q < n_chunks; q += nw * RPW) {
    const int64_t beg = cbeg[q], end = cend[q];
    T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int64_t e = beg;
    for (; e + 8 <= end; e += 8) {
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = __ldg(col + e + u);
      V2 z0[8], z1[8];
      T sv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const T* zr = zc + (int64_t)c[u] * KP;
        z0[u] = __ldg(reinterpret_cast<const V2*>(zr));
        z1[u] = __ldg(reinterpret_cast<const V2*>(zr + H2));
        if constexpr (sizeof(T) == 8) sv[u] = (T)__ldg(s + c[u]);
        else sv[u] = (T)__ldg(s32 + c[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = fma(sv[u], z0[u].x, a0);
        a1 = fma(sv[u], z0[u].y, a1);
        a2 = fma(sv[u], z1[u].x, a2);
        a3 = fma(sv[u], z1[u].y, a3);
      }
    }
    for (; e < end; ++e) {
      const int c = __ldg(col + e);
      const T* zr = zc + (int64_t)c * KP;
      const V2 z0 = __ldg(reinterpret_cast<const V2*>(zr));
      const V2 z1 = __ldg(reinterpret_cast<const V2*>(zr + H2));
      T sv;
      if constexpr (sizeof(T) == 8) sv = (T)__ldg(s + c);
      else sv = (T)__ldg(s32 + c);
      a0 = fma(sv, z0.x, a0);
      a1 = fma(sv, z0.y, a1);
      a2 = fma(sv, z1.x, a2);
      a3 = fma(sv, z1.y, a3);
    }
    T* o = scratch + q * 64 + 2 * l;
    o[0] = a0;
    o[1] = a1;
    o[H2] = a2;
    o[H2 + 1] = a3;
  }
}

template <typename T, int PHASE>
__global__ void k_heavy_finish(int64_t n_heavy, int KP, const int32_t* __restrict__ rows,
                               const int32_t* __restrict__ first, const T* __restrict__ scratch,
                               int64_t own_off, const double* __restrict__ s,
                               const float* __restrict__ s32, const T* __restrict__ Zg,
                               T* __restrict__ Y, const int* stop) {
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_heavy * KP;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = e / KP;
    const int c = (int)(e % KP);
    const int64_t i = rows[h];
    T acc = 0;
    if constexpr (PHASE == 2) acc = Y[i * KP + c];
    for (int q = first[h]; q < first[h + 1]; ++q) acc = acc + scratch[(int64_t)q * 64 + c];
    if constexpr (PHASE == 1) {
      Y[i * KP + c] = acc;
    } else {
      T si;
      if constexpr (sizeof(T) == 8) si = (T)s[own_off + i];
      else si = s32[own_off + i];
      Y[i * KP + c] = -Zg[(own_off + i) * KP + c] - si * acc;
    }
  }
}

static void launch_heavy(ofsc_dtype dt, int KP, int64_t own_off, const int64_t* row_ptr,
                         const int32_t* col, const double* s, const float* s32, const void* Zg,
                         void* Y, const int* stop, cudaStream_t st, int phase, const HeavyRows& hr) {
  (void)row_ptr;
  const int nbc = (int)std::min<int64_t>((hr.n_chunks * 32 + kThreads - 1) / kThreads,
                                         (int64_t)num_sms() * 8);
  const int nbf = (int)std::min<int64_t>((hr.n_rows * KP + 255) / 256, (int64_t)num_sms() * 8);
  OFSC_DISPATCH_KP(KP, {
    if (dt == OFSC_F64) {
      k_spmm_chunks<double, KPC><<<std::max(nbc, 1), kThreads, 0, st>>>(
          hr.n_chunks, hr.chunk_beg, hr.chunk_end, col, s, s32, (const double*)Zg,
          (double*)hr.scratch, stop);
    } else {
      k_spmm_chunks<float, KPC><<<std::max(nbc, 1), kThreads, 0, st>>>(
          hr.n_chunks, hr.chunk_beg, hr.chunk_end, col, s, s32, (const float*)Zg,
          (float*)hr.scratch, stop);
    }
  });
  OFSC_LAUNCH_CHECK();
#define OFSC_HF(TT, PH)                                                                           \
  k_heavy_finish<TT, PH><<<std::max(nbf, 1), 256, 0, st>>>(hr.n_rows, KP, hr.rows, hr.chunk_first, \
      (const TT*)hr.scratch, own_off, s, s32, (const TT*)Zg, (TT*)Y, stop)
  if (dt == OFSC_F64) {
    if (phase == 1) OFSC_HF(double, 1); else if (phase == 2) OFSC_HF(double, 2); else OFSC_HF(double, 0);
  } else {
    if (phase == 1) OFSC_HF(float, 1); else if (phase == 2) OFSC_HF(float, 2); else OFSC_HF(float, 0);
  }
#undef OFSC_HF
  OFSC_LAUNCH_CHECK();
}

__global__ void k_heavy_flags(int64_t n, const int64_t* row_ptr, int64_t thresh, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (row_ptr[i + 1] - row_ptr[i]) > thresh ? 1 : 0;
}

__global__ void k_iota_rows(int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

__global__ void k_row_bounds(int64_t nh, const int32_t* rows, const int64_t* row_ptr, int64_t* b,
                             int64_t* e) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nh;
       h += (int64_t)gridDim.x * blockDim.x) {
    b[h] = row_ptr[rows[h]];
    e[h] = row_ptr[rows[h] + 1];
  }
}

void HeavyRows::release() {
  if (rows) cudaDeviceSynchronize();   // pool frees below: no queued user left
  for (void* q : {(void*)rows, (void*)chunk_first, (void*)chunk_beg, (void*)chunk_end, scratch})
    dev_free(q);
  rows = nullptr;
  chunk_first = nullptr;
  chunk_beg = chunk_end = nullptr;
  scratch = nullptr;
  n_rows = n_chunks = 0;
  thresh = INT64_MAX;
}

void build_heavy(const int64_t* d_row_ptr, int64_t n_rows, HeavyRows& out, cudaStream_t st) {
  out.release();
  if (n_rows <= 0) return;
  const int64_t thresh = env_int("OFSC_HEAVY_THRESH", (int)kHeavyThresh);
  int* flag = nullptr;
  int32_t *iota = nullptr, *sel = nullptr;
  int64_t* nsel = nullptr;
  OFSC_CUDA(cudaMallocAsync(&flag, n_rows * sizeof(int), st));
  OFSC_CUDA(cudaMallocAsync(&iota, n_rows * sizeof(int32_t), st));
  OFSC_CUDA(cudaMallocAsync(&sel, n_rows * sizeof(int32_t), st));
  OFSC_CUDA(cudaMallocAsync(&nsel, sizeof(int64_t), st));
  const int nb = (int)std::min<int64_t>((n_rows + 255) / 256, (int64_t)num_sms() * 16);
  k_heavy_flags<<<nb, 256, 0, st>>>(n_rows, d_row_ptr, thresh, flag);
  k_iota_rows<<<nb, 256, 0, st>>>(n_rows, iota);
  OFSC_LAUNCH_CHECK();
  size_t tb = 0;
  OFSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, flag, sel, nsel, n_rows, st));
  void* tmp = nullptr;
  OFSC_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
  OFSC_CUDA(cub::DeviceSelect::Flagged(tmp, tb, iota, flag, sel, nsel, n_rows, st));
  int64_t nh = 0;
  OFSC_CUDA(cudaMemcpyAsync(&nh, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  OFSC_CUDA(cudaStreamSynchronize(st));
  if (nh > 0) {
    std::vector<int32_t> rows(nh);
    std::vector<int64_t> b(nh), e(nh);
    int64_t *db = nullptr, *de = nullptr;
    OFSC_CUDA(cudaMallocAsync(&db, nh * sizeof(int64_t), st));
    OFSC_CUDA(cudaMallocAsync(&de, nh * sizeof(int64_t), st));
    k_row_bounds<<<(int)std::min<int64_t>((nh + 255) / 256, 1024), 256, 0, st>>>(nh, sel, d_row_ptr,
                                                                               db, de);
    OFSC_LAUNCH_CHECK();
    OFSC_CUDA(cudaMemcpyAsync(rows.data(), sel, nh * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(b.data(), db, nh * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaMemcpyAsync(e.data(), de, nh * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    OFSC_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(db, st);
    cudaFreeAsync(de, st);
    std::vector<int32_t> first(nh + 1, 0);
    std::vector<int64_t> cb, ce;
    for (int64_t h = 0; h < nh; ++h) {
      first[h] = (int32_t)cb.size();
      for (int64_t x = b[h]; x < e[h]; x += kHeavyChunk) {
        cb.push_back(x);
        ce.push_back(std::min(e[h], x + kHeavyChunk));
      }
    }
    first[nh] = (int32_t)cb.size();
    out.thresh = thresh;
    out.n_rows = nh;
    out.n_chunks = (int64_t)cb.size();
    dev_alloc((void**)&out.rows, nh * sizeof(int32_t), st);
    dev_alloc((void**)&out.chunk_first, (nh + 1) * sizeof(int32_t), st);
    dev_alloc((void**)&out.chunk_beg, out.n_chunks * sizeof(int64_t), st);
    dev_alloc((void**)&out.chunk_end, out.n_chunks * sizeof(int64_t), st);
    dev_alloc((void**)&out.scratch, out.n_chunks * 64 * sizeof(double), st);
    OFSC_CUDA(cudaMemcpy(out.rows, rows.data(), nh * sizeof(int32_t), cudaMemcpyHostToDevice));
    OFSC_CUDA(cudaMemcpy(out.chunk_first, first.data(), (nh + 1) * sizeof(int32_t),
                         cudaMemcpyHostToDevice));
    OFSC_CUDA(cudaMemcpy(out.chunk_beg, cb.data(), out.n_chunks * sizeof(int64_t),
                         cudaMemcpyHostToDevice));
    OFSC_CUDA(cudaMemcpy(out.chunk_end, ce.data(), out.n_chunks * sizeof(int64_t),
                         cudaMemcpyHostToDevice));
  }
  cudaFreeAsync(flag, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(sel, st);
  cudaFreeAsync(nsel, st);
  cudaFreeAsync(tmp, st);
}

__global__ void k_gather_sval(int64_t nnz, const int32_t* col, const double* s, const float* s32,
                              double* sval, float* sval32) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    sval[e] = s[col[e]];
    sval32[e] = s32[col[e]];
  }
}

// packed stream: colpack[e] = col[e] | deg(col[e]) << 23; tables tab[d] = s of any
// node of degree d (every node of one degree has the same s bits: s = d^{-1/2} is a
// function of d), so s_j = tab[deg_j] reproduces the s_j of the other streams exactly
__global__ void k_pack_cols(int64_t nnz, const int32_t* col, const int64_t* row_ptr,
                            int32_t* colpack) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = col[e];
    const int64_t d = row_ptr[j + 1] - row_ptr[j];
    colpack[e] = j | (int32_t)((uint32_t)d << kPackShift);
  }
}
__global__ void k_deg_table(int64_t n, const int64_t* row_ptr, const double* s, const float* s32,
                            double* tab, float* tab32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = row_ptr[i + 1] - row_ptr[i];
    tab[d] = s[i];        // the same bits from every node of degree d
    tab32[d] = s32[i];
  }
}

void SvalStream::release() {
  if (sval || sval32 || colpack) cudaDeviceSynchronize();   // pool frees: no queued user left
  dev_free(sval);
  dev_free(sval32);
  dev_free(colpack);
  sval = nullptr;
  sval32 = nullptr;
  colpack = nullptr;
  mode = 0;
}

void build_sval(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* s, const float* s32, int64_t max_deg, SvalStream& out,
                cudaStream_t st) {
  out.release();
  // auto for graphs whose gathers mostly miss L2 (nnz >= 2e7; on L2-resident c3 an
  // extra stream cost 3 %).  OFSC_SPMM_SVAL: 0 off (s_j gathered by column id),
  // 1 per-nonzero s_j (8 extra bytes per nonzero; c4 SpMM 5.6 -> 5.3 ms in round 1),
  // 2 packed (column | degree) stream + per-degree table (no extra bytes; needs
  // n <= 2^23 and max degree < 2^9).  Default: 2 when it fits and nnz >= 1e7,
  // else 1 for nnz >= 2e7.
  const int env = env_int("OFSC_SPMM_SVAL", -1);
  const bool fits = n <= ((int64_t)1 << kPackShift) && max_deg < (1 << (32 - kPackShift));
  // measured (profiles/r02/spmm_sval_ab*.jsonl): packed c4 -4 %, c6 -4 %, c5 (16M
  // nonzeros) -2.5 %, neutral to +1 % on the L2-resident c1-c3
  int mode = env >= 0 ? env : (fits ? (nnz >= 10000000 ? 2 : 0) : (nnz >= 20000000 ? 1 : 0));
  if (mode == 2 && !fits) mode = 1;
  if (nnz <= 0 || mode <= 0) return;
  if (mode == 1) {
    dev_alloc((void**)&out.sval, nnz * sizeof(double), st);
    dev_alloc((void**)&out.sval32, nnz * sizeof(float), st);
    k_gather_sval<<<num_sms() * 16, 256, 0, st>>>(nnz, col, s, s32, out.sval, out.sval32);
  } else {
    dev_alloc((void**)&out.colpack, nnz * sizeof(int32_t), st);
    dev_alloc((void**)&out.sval, (max_deg + 1) * sizeof(double), st);
    dev_alloc((void**)&out.sval32, (max_deg + 1) * sizeof(float), st);
    OFSC_CUDA(cudaMemsetAsync(out.sval, 0, (max_deg + 1) * sizeof(double), st));
    OFSC_CUDA(cudaMemsetAsync(out.sval32, 0, (max_deg + 1) * sizeof(float), st));
    k_pack_cols<<<num_sms() * 16, 256, 0, st>>>(nnz, col, row_ptr, out.colpack);
    k_deg_table<<<num_sms() * 8, 256, 0, st>>>(n, row_ptr, s, s32, out.sval, out.sval32);
  }
  OFSC_LAUNCH_CHECK();
  out.mode = mode;
}

// Default column window of the SpMM passes (see k_spmm).
int spmm_col_window(ofsc_dtype, int KP) { return KP; }

int spmm_grid(int64_t n_local) {  // resident CTAs (3 per SM) for the chunked schedule
  const int64_t warps = (n_local + 1) / 2;
  int64_t b = (warps * 32 + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)num_sms() * env_int("OFSC_SPMM_CTAS_PER_SM", 3);
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

void launch_spmm(ofsc_dtype dt, int KP, int64_t n_local, int64_t own_off, const int64_t* row_ptr,
                 const int32_t* col, const double* s, const float* s32, const void* Zg, void* Y,
                 const int* stop, cudaStream_t st, const int32_t* cid, const int64_t* cstart,
                 unsigned long long* ctr, int phase, const HeavyRows* heavy,
                 const SvalStream* svs, int64_t nnz) {
  const int svm = (svs && phase == 0) ? svs->mode : 0;
  const void* sval = svm ? (dt == OFSC_F64 ? (const void*)svs->sval : (const void*)svs->sval32)
                         : nullptr;
  if (svm == 2) col = svs->colpack;
  const bool hv = heavy && heavy->n_rows > 0;
  const int64_t hth = hv ? heavy->thresh : INT64_MAX;
  // cid / cstart: community layout of reordered graphs (p == 1), for the L2 hints.
  const int hint = (cid && cstart && own_off == 0) ? env_int("OFSC_SPMM_HINT", 0) : 0;
  const int nb = spmm_grid(n_local);
  // rows per work grab (tuning knob): 4 at KP = 64 (c4 5.26 -> 5.21 ms, c6 1.70 -> 1.67),
  // 8 otherwise (c5, KP = 48: 0.776 vs 0.785 ms)
  const int ch = env_int("OFSC_SPMM_CHUNK", KP == 64 ? 4 : kSpmmChunk);
  int cw = env_int("OFSC_SPMM_CW", spmm_col_window(dt, KP));  // columns per pass (tuning knob)
  if (cw != 16 && cw != 32) cw = KP;
  if (phase) cw = KP;                       // split (multi-GPU) passes use whole rows
  if (KP % cw) cw = KP;
  const int passes = KP / cw;
  // L2 prefetch of the neighbour rows beyond the 8 the registers hold (PF = 2: the
  // row start prefetches neighbours 8..8+LPR-1, each batch the rows 16..23 ahead;
  // PF = 1: next batch only; PF = 3: + the next row's first LPR neighbours).
  // Measured (profiles/r02/spmm_pf_sweep.jsonl, SpMM ms, PF 0 / 1 / 2 / 3):
  //   c4 5.30 / 5.19 / 4.99 / 6.10   c5 0.792 / 0.777 / 0.743 / 0.771
  //   c6 1.70 / 1.85 / 1.78 / 2.01   c3 0.150 / 0.154 / 0.150 / 0.171
  // i.e. it pays where the gathered operand is well beyond L2 and rows are short
  // (c4, c5: most neighbour rows miss L2), and costs where the community windows
  // stay L2-resident (c3) or long rows already keep many loads in flight (c6, avg
  // degree 47).  Default: PF = 2 when N KP w > 256 MB and nnz / N <= 32, else 0;
  // OFSC_SPMM_PF overrides (s_j-stream graphs), OFSC_SPMM_PF_SMALL (the others).
  const int64_t gather_mb = n_local * KP * (dt == OFSC_F64 ? 8 : 4) >> 20;
  const bool short_rows = n_local > 0 && nnz >= 0 && nnz <= 32 * n_local;
  const int pf_auto = (gather_mb > 256 && short_rows) ? 2 : 0;
  const int pfe = env_int("OFSC_SPMM_PF", pf_auto);
  const int pfn = env_int("OFSC_SPMM_PF_SMALL", pf_auto);
  // neighbour rows in flight per row group: 8 at 3 CTAs/SM (80 registers), 6 at 4 CTAs
  // (64 registers: same loads in flight, a third more warps), 4 at 5 (spills).  Measured
  // on the packed-stream path (profiles/r02/spmm_nif_ab.jsonl, SpMM ms, NIF 8 / 6 / 4):
  // c4 4.72-4.91 / 4.68-4.79 / 5.12-5.18, c5 0.722 / 0.698 / 0.739, c6 neutral.
  const int nif = env_int("OFSC_SPMM_NIF", svm == 2 ? 6 : 8);
  const int nb4 = (int)std::min<int64_t>((int64_t)num_sms() * 4, std::max<int64_t>(nb, 1) * 4 / 3 + 1);
  const int nb5 = (int)std::min<int64_t>((int64_t)num_sms() * 5, std::max<int64_t>(nb, 1) * 5 / 3 + 1);
  // a PDL launch (the iteration's SpMM right after C4) must not be preceded by a memset:
  // there k_beta has zeroed the counters (IterParams::spmm_ctr)
  const bool pdl_first = pdl_take();
  // static interleaved row assignment (no global counter) when the gathered operand is
  // below OFSC_SPMM_STATIC_KB kilobytes (default 16 MB): a graph that small stays in L2
  // whatever the row order, and the counter costs an atomic round trip per chunk.
  // Measured (profiles/r02/spmm_static_ab.jsonl, same sums): c1 32.6 -> 31.2 us, c2
  // 70.0 -> 68.9 us per iteration; at c3 (102 MB, ~ the L2) the in-order window is
  // needed (0.547 -> 0.605 ms static), so it keeps the counter.
  {
    const int64_t static_kb = env_int("OFSC_SPMM_STATIC_KB", 16384);
    const int64_t op_kb = (n_local + own_off) * KP * (dt == OFSC_F64 ? 8 : 4) >> 10;
    if (static_kb > 0 && op_kb < static_kb && phase == 0) ctr = nullptr;
  }
  if (ctr && !pdl_first) OFSC_CUDA(cudaMemsetAsync(ctr, 0, passes * sizeof(unsigned long long), st));
  for (int ps = 0; ps < passes; ++ps) {
    const bool pdl = pdl_first && ps == 0;
    unsigned long long* c = ctr ? ctr + ps : nullptr;
    const int c0 = ps * cw;
#define OFSC_SPMM_LAUNCH_N(CWC, H, PH, SVV, PFF, NN, NBB)                                       \
    if (dt == OFSC_F64)                                                                         \
      launch_k(k_spmm<double, KPC, CWC, H, PH, SVV, PFF, NN>, dim3(NBB), dim3(kThreads), 0, st, \
               pdl, n_local, own_off, row_ptr, col, s, s32, (const double*)Zg, (double*)Y,       \
               stop, c, ch, c0, cid, cstart, hth, (const double*)sval);                          \
    else                                                                                        \
      launch_k(k_spmm<float, KPC, CWC, H, PH, SVV, PFF, NN>, dim3(NBB), dim3(kThreads), 0, st,  \
               pdl, n_local, own_off, row_ptr, col, s, s32, (const float*)Zg, (float*)Y, stop,   \
               c, ch, c0, cid, cstart, hth, (const float*)sval);
#define OFSC_SPMM_LAUNCH_F(CWC, H, PH, SVV, PFF) OFSC_SPMM_LAUNCH_N(CWC, H, PH, SVV, PFF, 8, nb)
#define OFSC_SPMM_LAUNCH_S(CWC, H, PH, SVV) OFSC_SPMM_LAUNCH_F(CWC, H, PH, SVV, 0)
#define OFSC_SPMM_LAUNCH_P(CWC, H, PH) OFSC_SPMM_LAUNCH_S(CWC, H, PH, 0)
#define OFSC_SPMM_LAUNCH_H(CWC, H) OFSC_SPMM_LAUNCH_P(CWC, H, 0)
#define OFSC_SPMM_LAUNCH(CWC) \
    if (hint) { OFSC_SPMM_LAUNCH_H(CWC, 1) } else { OFSC_SPMM_LAUNCH_H(CWC, 0) }
    OFSC_DISPATCH_KP(KP, {
      if (svm == 2 && cw == KPC && !hint && nif == 6) {
        if (pfe == 2) { OFSC_SPMM_LAUNCH_N(KPC, 0, 0, 2, 2, 6, nb4) }
        else { OFSC_SPMM_LAUNCH_N(KPC, 0, 0, 2, 0, 6, nb4) }
      }
      else if (svm == 2 && cw == KPC && !hint && nif == 4) {
        if (pfe == 2) { OFSC_SPMM_LAUNCH_N(KPC, 0, 0, 2, 2, 4, nb5) }
        else { OFSC_SPMM_LAUNCH_N(KPC, 0, 0, 2, 0, 4, nb5) }
      }
      else if (svm == 2 && cw == KPC && !hint) {
        if (pfe == 2) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 2, 2) }
        else { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 2, 0) }
      }
      else if (svm == 1 && cw == KPC && !hint) {
        if (pfe == 3) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 1, 3) }
        else if (pfe == 2) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 1, 2) }
        else if (pfe == 1) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 1, 1) }
        else { OFSC_SPMM_LAUNCH_S(KPC, 0, 0, 1) }
      }
      else if (phase == 1) { OFSC_SPMM_LAUNCH_P(KPC, 0, 1) }
      else if (phase == 2) { OFSC_SPMM_LAUNCH_P(KPC, 0, 2) }
      else if (cw == KPC && !hint && pfn > 0) {     // gathered s_j + L2 prefetch
        if (pfn == 3) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 0, 3) }
        else if (pfn == 2) { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 0, 2) }
        else { OFSC_SPMM_LAUNCH_F(KPC, 0, 0, 0, 1) }
      }
      else if (cw == KPC) { OFSC_SPMM_LAUNCH(KPC) }
      else if (cw == 32) { if constexpr (KPC % 32 == 0) { OFSC_SPMM_LAUNCH(32) } }
      else { if constexpr (KPC % 16 == 0) { OFSC_SPMM_LAUNCH(16) } }
    });
#undef OFSC_SPMM_LAUNCH
#undef OFSC_SPMM_LAUNCH_H
#undef OFSC_SPMM_LAUNCH_P
#undef OFSC_SPMM_LAUNCH_S
#undef OFSC_SPMM_LAUNCH_F
#undef OFSC_SPMM_LAUNCH_N
    OFSC_LAUNCH_CHECK();
  }
  if (hv) launch_heavy(dt, KP, own_off, row_ptr, col, s, s32, Zg, Y, stop, st, phase, *heavy);
}

void launch_spmm_then_gram(ofsc_dtype dt, int KP, int64_t n_local, int64_t own_off,
                      const int64_t* row_ptr, const int32_t* col, const double* s,
                      const float* s32, const void* Zg, const void* Xown, void* Y, double* part,
                      int mode, const int* stop, int nblk, cudaStream_t st,
                      const HeavyRows* heavy, unsigned long long* ctr, const SvalStream* svs,
                      int64_t nnz) {
  launch_spmm(dt, KP, n_local, own_off, row_ptr, col, s, s32, Zg, Y, stop, st, nullptr, nullptr,
              ctr, 0, heavy, svs, nnz);
  if (part) {
    const size_t es = dt == OFSC_F64 ? 8 : 4;
    const void* Zown = (const char*)Zg + (size_t)own_off * KP * es;
    launch_gram_stream(dt, KP, n_local, Zown, mode == 0 ? Xown : nullptr, Y, part, mode, stop,
                       nblk, st);
  }
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

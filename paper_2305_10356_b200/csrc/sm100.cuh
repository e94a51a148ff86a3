// sm_100a building blocks: TMA bulk copies (cp.async.bulk) with mbarrier
// completion, and the fp64 tensor-core MMA (mma.sync m8n8k4 f64 -> DMMA.8x8x4;
// tcgen05 has no f64 kind, measured 37.1 TF/s vs 33.4 for DFMA, profiles/r01).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ofsc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- programmatic dependent launch (PDL) ----------------------------------------
// A kernel launched with programmatic stream serialization may be scheduled while
// its predecessor drains; pdl_wait() (griddepcontrol.wait) blocks until the
// predecessor grid has completed and its memory is visible, so every kernel of the
// PDL chain calls it before touching anything a predecessor wrote.  Without the
// launch attribute both are no-ops.  pdl_trigger() lets the dependent be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier --------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// named barrier over `count` threads (a subset of the CTA, e.g. the producer warps)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// ---- TMA bulk copies (1-D, 16-byte aligned, size multiple of 16) -------------
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy smem writes -> visible to the async proxy (TMA store reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- cp.async (LDGSTS): per-thread global -> shared copies, zero-filled
// beyond src_bytes; completion by commit / wait groups --------------------------
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc, int src_bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(gsrc), "n"(BYTES),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- fp64 MMA: D(8x8) += A(8x4) B(4x8) --------------------------------------
// Fragments (PTX ISA, m8n8k4 .f64): gid = lane >> 2, tig = lane & 3;
//   a = A[gid][tig], b = B[tig][gid], d0 = D[gid][2 tig], d1 = D[gid][2 tig + 1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Warp tiling of a KP x KP output into 8x8 MMA blocks for 4 warps:
// warp wp (0..3) owns blocks ib in [IB0, IB0 + BI), jb in [JB0, JB0 + BJ).
template <int KP>
struct WarpTiling;
template <>
struct WarpTiling<16> {
  static constexpr int BI = 1, BJ = 1;
  __device__ static int ib0(int wp) { return wp >> 1; }
  __device__ static int jb0(int wp) { return wp & 1; }
};
template <>
struct WarpTiling<32> {
  static constexpr int BI = 1, BJ = 4;
  __device__ static int ib0(int wp) { return wp; }
  __device__ static int jb0(int) { return 0; }
};
template <>
struct WarpTiling<48> {
  static constexpr int BI = 3, BJ = 3;
  __device__ static int ib0(int wp) { return 3 * (wp >> 1); }
  __device__ static int jb0(int wp) { return 3 * (wp & 1); }
};
template <>
struct WarpTiling<64> {
  static constexpr int BI = 2, BJ = 8;
  __device__ static int ib0(int wp) { return 2 * wp; }
  __device__ static int jb0(int) { return 0; }
};

// Two k x k Gram products over a tile of `rows` rows held in padded smem
// (row stride LD = KP + 4 doubles: the 4-row x 8-column fragment reads hit
// every bank exactly twice, i.e. the 2-wavefront minimum):
//   acc(prod 0) += L1^T R1 (warps 0-3),  acc(prod 1) += L2^T R2 (warps 4-7).
template <int KP>
struct DmmaGram {
  static constexpr int LD = KP + 4;
  using WT = WarpTiling<KP>;
  static constexpr int BI = WT::BI, BJ = WT::BJ;
  double d[BI][BJ][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < BI; ++i)
#pragma unroll
      for (int j = 0; j < BJ; ++j) d[i][j][0] = d[i][j][1] = 0.0;
  }
  // rows: multiple of 4 (tiles are zero-padded to that); 8 warps
  __device__ __forceinline__ void accumulate(const double* L1, const double* R1, const double* L2,
                                             const double* R2, int rows, int warp, int lane) {
    const int gid = lane >> 2, tig = lane & 3, wp = warp & 3;
    const double* L = (warp >> 2) ? L2 : L1;
    const double* R = (warp >> 2) ? R2 : R1;
    const double* Lc = L + WT::ib0(wp) * 8 + gid;
    const double* Rc = R + WT::jb0(wp) * 8 + gid;
    for (int r0 = 0; r0 < rows; r0 += 4) {
      const int rr = (r0 + tig) * LD;
      double a[BI], b[BJ];
#pragma unroll
      for (int i = 0; i < BI; ++i) a[i] = Lc[rr + i * 8];
#pragma unroll
      for (int j = 0; j < BJ; ++j) b[j] = Rc[rr + j * 8];
#pragma unroll
      for (int i = 0; i < BI; ++i)
#pragma unroll
        for (int j = 0; j < BJ; ++j) dmma(d[i][j][0], d[i][j][1], a[i], b[j]);
    }
  }
  // out[prod][i][j] (row-major KP x KP each); prod = warp >> 2
  __device__ __forceinline__ void store(double* out, int warp, int lane) const {
    const int gid = lane >> 2, tig = lane & 3, wp = warp & 3;
    double* o = out + (warp >> 2) * KP * KP;
#pragma unroll
    for (int i = 0; i < BI; ++i)
#pragma unroll
      for (int j = 0; j < BJ; ++j) {
        double* q = o + ((WT::ib0(wp) + i) * 8 + gid) * KP + (WT::jb0(wp) + j) * 8 + 2 * tig;
        q[0] = d[i][j][0];
        q[1] = d[i][j][1];
      }
  }
};

// KP = 64 with a symmetric first product (Q = V^T V, T = V^T A V, M = X^T X):
// only its 36 upper 8x8 blocks are computed (mirrored on store), and the 100
// tiles are balanced over the 8 warps (12 or 13 each):
//   warps 0-3:      product 1, block rows {2w, 2w+1} x block cols 0..5   (12 tiles)
//   warps 4+q:      product 0, block rows q (cols q..7) and 7-q (cols 7-q..7) (9 tiles)
//                   + product 1, block rows {2q, 2q+1} x cols {6, 7}          (4 tiles)
struct DmmaGramSym64 {
  static constexpr int KP = 64, LD = 68;
  double d[13][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int u = 0; u < 13; ++u) d[u][0] = d[u][1] = 0.0;
  }
  template <int Q>
  __device__ __forceinline__ void sym_step(const double* L0, const double* R0, const double* L1,
                                           const double* R1, int rr, int gid) {
    const double a0 = L0[rr + Q * 8 + gid];
    const double a1 = L0[rr + (7 - Q) * 8 + gid];
    constexpr int J0 = Q < 7 - Q ? Q : 7 - Q;
    double b[8];
#pragma unroll
    for (int j = J0; j < 8; ++j) b[j] = R0[rr + j * 8 + gid];
#pragma unroll
    for (int j = Q; j < 8; ++j) dmma(d[j - Q][0], d[j - Q][1], a0, b[j]);
#pragma unroll
    for (int j = 7 - Q; j < 8; ++j) dmma(d[(8 - Q) + j - (7 - Q)][0], d[(8 - Q) + j - (7 - Q)][1], a1, b[j]);
    const double c0 = L1[rr + (2 * Q) * 8 + gid], c1 = L1[rr + (2 * Q + 1) * 8 + gid];
    const double e6 = R1[rr + 6 * 8 + gid], e7 = R1[rr + 7 * 8 + gid];
    dmma(d[9][0], d[9][1], c0, e6);
    dmma(d[10][0], d[10][1], c0, e7);
    dmma(d[11][0], d[11][1], c1, e6);
    dmma(d[12][0], d[12][1], c1, e7);
  }
  __device__ __forceinline__ void accumulate(const double* L0, const double* R0, const double* L1,
                                             const double* R1, int rows, int warp, int lane) {
    const int gid = lane >> 2, tig = lane & 3;
    if (warp < 4) {
      for (int r0 = 0; r0 < rows; r0 += 4) {
        const int rr = (r0 + tig) * LD;
        const double a0 = L1[rr + (2 * warp) * 8 + gid], a1 = L1[rr + (2 * warp + 1) * 8 + gid];
        double b[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) b[j] = R1[rr + j * 8 + gid];
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          dmma(d[j][0], d[j][1], a0, b[j]);
          dmma(d[6 + j][0], d[6 + j][1], a1, b[j]);
        }
      }
    } else {
      const int q = warp - 4;
      for (int r0 = 0; r0 < rows; r0 += 4) {
        const int rr = (r0 + tig) * LD;
        switch (q) {
          case 0: sym_step<0>(L0, R0, L1, R1, rr, gid); break;
          case 1: sym_step<1>(L0, R0, L1, R1, rr, gid); break;
          case 2: sym_step<2>(L0, R0, L1, R1, rr, gid); break;
          default: sym_step<3>(L0, R0, L1, R1, rr, gid); break;
        }
      }
    }
  }
  // out[0] = product 0 (full, mirrored), out[1] = product 1 (row-major 64 x 64 each)
  __device__ __forceinline__ void put(double* o, int ib, int jb, int gid, int tig, const double* v) const {
    double* q = o + (ib * 8 + gid) * KP + jb * 8 + 2 * tig;
    q[0] = v[0];
    q[1] = v[1];
  }
  __device__ __forceinline__ void put_sym(double* o, int ib, int jb, int gid, int tig,
                                          const double* v) const {
    put(o, ib, jb, gid, tig, v);
    if (ib != jb) {   // mirror: (jb*8 + 2tig + h, ib*8 + gid)
      o[(jb * 8 + 2 * tig) * KP + ib * 8 + gid] = v[0];
      o[(jb * 8 + 2 * tig + 1) * KP + ib * 8 + gid] = v[1];
    }
  }
  template <int Q>
  __device__ __forceinline__ void store_q(double* out, int gid, int tig) const {
#pragma unroll
    for (int j = Q; j < 8; ++j) put_sym(out, Q, j, gid, tig, d[j - Q]);
#pragma unroll
    for (int j = 7 - Q; j < 8; ++j) put_sym(out, 7 - Q, j, gid, tig, d[(8 - Q) + j - (7 - Q)]);
    double* o1 = out + KP * KP;
    put(o1, 2 * Q, 6, gid, tig, d[9]);
    put(o1, 2 * Q, 7, gid, tig, d[10]);
    put(o1, 2 * Q + 1, 6, gid, tig, d[11]);
    put(o1, 2 * Q + 1, 7, gid, tig, d[12]);
  }
  __device__ __forceinline__ void store(double* out, int warp, int lane) const {
    const int gid = lane >> 2, tig = lane & 3;
    if (warp < 4) {
      double* o1 = out + KP * KP;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        put(o1, 2 * warp, j, gid, tig, d[j]);
        put(o1, 2 * warp + 1, j, gid, tig, d[6 + j]);
      }
    } else {
      switch (warp - 4) {
        case 0: store_q<0>(out, gid, tig); break;
        case 1: store_q<1>(out, gid, tig); break;
        case 2: store_q<2>(out, gid, tig); break;
        default: store_q<3>(out, gid, tig); break;
      }
    }
  }
};

// Gram accumulator for a tile width: the symmetric-aware one at KP = 64.
template <int KP>
struct GramSel {
  using type = DmmaGram<KP>;
};
template <>
struct GramSel<64> {
  using type = DmmaGramSym64;
};

}  // namespace ofsc

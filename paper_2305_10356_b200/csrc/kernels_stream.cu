// Streaming row kernels of the iteration, TMA-pipelined (sm_100a):
//   C3  k_update_direction: X += alpha V, AX += alpha AV (Alg. 2 l.12, applied
//       lazily), G = g_m(X) (eq:gradientf1/g1/f2/g2) and the column
//       dots of Alg. 2 l.9;
//   C4  k_direction_gram: V = -G + beta Vp (Alg. 2 l.10) fused with the Grams
//       Q = V^T V, P = V^T X of the line-search cubics.
// Row tiles (TR rows x KP columns) are contiguous in HBM, so each operand tile
// is one 1-D TMA bulk copy (cp.async.bulk) into an S-stage shared-memory ring
// completed on an mbarrier; results leave through TMA bulk stores from the same
// stage buffers.  The N x k . k x k products and the Grams run on the fp64
// tensor path (mma.sync m8n8k4 f64 = DMMA.8x8x4) from padded smem copies.
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace ofsc {

template <typename T>
__device__ __forceinline__ double rndT(double v) { return (double)(T)v; }

constexpr int kSTR = 16;   // rows per streamed tile
constexpr int kSST = 3;    // pipeline stages
// warp-specialised Gram kernels (C4, C2b)
constexpr int kGWS_NS = 3;          // TMA stages
constexpr int kGWS_NP = 2;          // padded tiles
constexpr int kGWS_THREADS = 384;   // 8 consumer + 4 producer warps

template <typename T, int KP>
struct StreamTile {
  static constexpr int LD = KP + 4;                                // padded double stride
  static constexpr uint32_t ARR = kSTR * KP * sizeof(T);           // bytes of one full tile array
};

// ---------------------------------------------------------------------------
// C3
// ---------------------------------------------------------------------------
// C3 tiling: warp w < KP/8 owns output column block cb = w for both 8-row blocks
// of the 16-row tile; its DMMA B-fragments of M (and W) -- 16 k-steps -- stay in
// registers for the whole kernel, so shared memory holds only the 2-stage TMA
// ring and the padded X', AX' tile (2 CTAs per SM).
constexpr int kC3Stages = 2;

// TR rows per tile, NS TMA stages (default 16 x 2; k_update_direction also has an
// 8-row x 4-stage form, A/B knob OFSC_C3_TR8: the same bytes of ring in flight, each
// stage released after half the work)
template <typename T, int KP, int METHOD, int TR = kSTR, int NS = kC3Stages>
struct C3Smem {
  static constexpr int LD = KP + 4;
  static constexpr size_t xp = (size_t)TR * LD * 8;
  static constexpr size_t arr = (size_t)TR * KP * sizeof(T);
  static constexpr size_t stage = 5 * arr;                          // X, AX, V, AV, G
  static constexpr size_t bytes = 2 * xp + NS * stage + KP * 8 + NS * 8;
};

template <typename T, int KP, int METHOD, int TR = kSTR, int NS = kC3Stages>
__global__ void __launch_bounds__(kThreads, 2)
k_update_direction(IterParams p, int apply_update) {
  using S = C3Smem<T, KP, METHOD, TR, NS>;
  constexpr int LD = S::LD;
  constexpr int SUB = kSTR / TR;                 // TR-row tiles per 16-row tile
  constexpr int RB = TR / 8;                     // 8-row DMMA blocks per tile
  constexpr bool TRI = (METHOD == OFSC_TRIOFM_F1 || METHOD == OFSC_TRIOFM_F2);
  constexpr bool F1 = (METHOD == OFSC_OFM_F1 || METHOD == OFSC_TRIOFM_F1);
  constexpr int NB = KP / 8;
  constexpr int KS = KP / 4;                     // DMMA k-steps
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* Xp = (double*)smraw;
  double* AXp = Xp + TR * LD;
  unsigned char* stg = smraw + 2 * S::xp;
  double* s_alpha = (double*)(stg + NS * S::stage);
  uint64_t* bar = (uint64_t*)(s_alpha + KP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t ntiles = (p.n_local + kSTR - 1) / kSTR;
  // the CTA's it-th tile: part it % SUB of its (it / SUB)-th 16-row tile, so every
  // thread visits the rows (and accumulates its column dots) in the same order for
  // any TR: the results are bitwise those of the 16-row form
  auto tile_row0 = [&](int64_t it) -> int64_t {
    const int64_t t16 = blockIdx.x + (it / SUB) * (int64_t)gridDim.x;
    return t16 < ntiles ? t16 * kSTR + (it % SUB) * TR : INT64_MAX;
  };
  T* gX = (T*)p.X;
  T* gAX = (T*)p.AX;
  T* gG = (T*)p.G;
  const T* gV = (const T*)p.V;
  const T* gAV = (const T*)p.AV;
  auto arr = [&](int st, int a) { return (T*)(stg + st * S::stage + a * S::arr); };  // 0 X,1 AX,2 V,3 AV,4 G
  auto issue = [&](int st, int64_t row0) {
    const int rows = (int)imin64(TR, p.n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&bar[st], (apply_update ? 5u : 3u) * b);
    const int64_t off = row0 * KP;
    bulk_g2s(arr(st, 0), gX + off, b, &bar[st]);
    bulk_g2s(arr(st, 1), gAX + off, b, &bar[st]);
    if (apply_update) {
      bulk_g2s(arr(st, 2), gV + off, b, &bar[st]);
      bulk_g2s(arr(st, 3), gAV + off, b, &bar[st]);
    }
    bulk_g2s(arr(st, 4), gG + off, b, &bar[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  if (tid < KP) s_alpha[tid] = apply_update ? p.alpha[tid] : 0.0;
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < NS; ++s) {
      const int64_t r0 = tile_row0(s);
      if (r0 < p.n_local) issue(s, r0);
    }
  // register-resident B fragments: B[k][n] = M[4 kk + tig][cb*8 + gid] (triu for TriOFM)
  const bool mma_warp = warp < NB;
  const int cb = mma_warp ? warp : 0;
  double bm[KS], bw[F1 ? 1 : KS];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int j = 4 * kk + tig, c = cb * 8 + gid;
    const bool keep = !TRI || j <= c;            // triu keeps the diagonal (R15)
    bm[kk] = keep ? p.M[j * KP + c] : 0.0;
    if (!F1) bw[kk] = keep ? p.W[j * KP + c] : 0.0;
  }
  double gg[2] = {0.0, 0.0}, dg[2] = {0.0, 0.0};
  for (int64_t it = 0;; ++it) {
    const int64_t row0 = tile_row0(it);
    if (row0 >= p.n_local) break;
    const int st = (int)(it % NS);
    const int rows = (int)imin64(TR, p.n_local - row0);
    mbar_wait(&bar[st], (uint32_t)((it / NS) & 1));
    T* sX = arr(st, 0);
    T* sAX = arr(st, 1);
    const T* sV = arr(st, 2);
    const T* sAV = arr(st, 3);
    T* sG = arr(st, 4);
    // phase A: X' = X + alpha V, AX' = AX + alpha AV (rounded to storage), padded copies
    for (int e = tid; e < TR * KP; e += kThreads) {
      const int r = e / KP, c = e % KP;
      double x = 0.0, ax = 0.0;
      if (r < rows) {
        x = (double)sX[e];
        ax = (double)sAX[e];
        if (apply_update) {
          x = rndT<T>(fma(s_alpha[c], (double)sV[e], x));
          ax = rndT<T>(fma(s_alpha[c], (double)sAV[e], ax));
          sX[e] = (T)x;
          sAX[e] = (T)ax;
        }
      }
      Xp[r * LD + c] = x;
      AXp[r * LD + c] = ax;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0 && apply_update) {
      const uint32_t b = (uint32_t)rows * KP * sizeof(T);
      bulk_s2g(gX + row0 * KP, sX, b);
      bulk_s2g(gAX + row0 * KP, sAX, b);
      bulk_commit();
    }
    if (mma_warp) {
      // phase B: G tile column block cb = f(X' M, X' W, AX' M) on DMMA (both row blocks)
      double a1[RB][2], a2[RB][2];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) a1[rb][0] = a1[rb][1] = a2[rb][0] = a2[rb][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        // TriOFM: triu(M), triu(W) vanish below the diagonal, so the k-steps whose rows
        // j = 4kk..4kk+3 all exceed this warp's columns 8cb..8cb+7 contribute exact
        // zeros: skipped (warp-uniform), half of the products on average
        if (TRI && 4 * kk > 8 * cb + 7) continue;
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          const int o = (rb * 8 + gid) * LD + 4 * kk + tig;
          const double xa = Xp[o];
          if (F1) {
            dmma(a1[rb][0], a1[rb][1], xa, bm[kk]);           // X M (or X triu M)
          } else {
            const double aa = AXp[o];
            dmma(a1[rb][0], a1[rb][1], xa, bw[kk]);           // X W (or X triu W)
            dmma(a2[rb][0], a2[rb][1], aa, bm[kk]);           // AX M (or AX triu M)
          }
        }
      }
      // phase C: G, column dots, in-place store into the stage's G tile
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        const int r = rb * 8 + gid;
        if (r < rows) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = cb * 8 + 2 * tig + h;
            const double ax = AXp[r * LD + c];
            double g;
            // explicit roundings: every C3 variant computes the same bits
            if (METHOD == OFSC_OFM_F1) g = fma(4.0, a1[rb][h], 4.0 * ax);
            else if (METHOD == OFSC_TRIOFM_F1) g = __dadd_rn(ax, a1[rb][h]);
            else if (METHOD == OFSC_OFM_F2) g = fma(-2.0, a2[rb][h], fma(-2.0, a1[rb][h], 4.0 * ax));
            else g = __dadd_rn(__dadd_rn(2.0 * ax, -a2[rb][h]), -a1[rb][h]);
            g = rndT<T>(g);
            const double gp = (double)sG[r * KP + c];
            sG[r * KP + c] = (T)g;
            gg[h] = fma(g, g, gg[h]);
            dg[h] = fma(g - gp, g, dg[h]);
          }
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(gG + row0 * KP, sG, (uint32_t)rows * KP * sizeof(T));
      bulk_commit();
      const int64_t nxt = tile_row0(it + NS);
      if (nxt < p.n_local) {
        bulk_wait_read_all();                     // stage st no longer read by the stores
        issue(st, nxt);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
  // column partials: lanes of one tig hold the same two columns -> reduce over gid
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      gg[h] += __shfl_xor_sync(0xffffffffu, gg[h], o);
      dg[h] += __shfl_xor_sync(0xffffffffu, dg[h], o);
    }
  if (mma_warp && gid == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = cb * 8 + 2 * tig + h;
      p.part_cols[(int64_t)blockIdx.x * 2 * KP + c] = gg[h];
      p.part_cols[(int64_t)blockIdx.x * 2 * KP + KP + c] = dg[h];
    }
  }
}

// C3, warp-specialised: the same 8 compute warps and arithmetic as
// k_update_direction (bitwise identical results), plus a 9th warp that owns the
// TMA traffic.  The compute warps hand each stage over on mbarriers (phase A done:
// X', AX' may be stored; phase C done: G may be stored) and never wait for the
// stores' shared-memory reads -- the producer waits for those and refills the
// stage, so the store-read latency leaves the compute warps' critical path.
constexpr int kC3WsThreads = kThreads + 32;

template <typename T, int KP, int METHOD>
struct C3WsSmem {
  static constexpr size_t base = C3Smem<T, KP, METHOD>::bytes;
  static constexpr size_t bytes = base + 2 * kC3Stages * 8;          // + adone, cdone barriers
};

template <typename T, int KP, int METHOD>
__global__ void __launch_bounds__(kC3WsThreads, 2)
k_update_direction_ws(IterParams p, int apply_update) {
  using S = C3Smem<T, KP, METHOD>;
  constexpr int LD = S::LD;
  constexpr int NS = kC3Stages;
  constexpr bool TRI = (METHOD == OFSC_TRIOFM_F1 || METHOD == OFSC_TRIOFM_F2);
  constexpr bool F1 = (METHOD == OFSC_OFM_F1 || METHOD == OFSC_TRIOFM_F1);
  constexpr int NB = KP / 8;
  constexpr int KS = KP / 4;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* Xp = (double*)smraw;
  double* AXp = Xp + kSTR * LD;
  unsigned char* stg = smraw + 2 * S::xp;
  double* s_alpha = (double*)(stg + NS * S::stage);
  uint64_t* full = (uint64_t*)(s_alpha + KP);
  uint64_t* adone = full + NS;
  uint64_t* cdone = adone + NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t ntiles = (p.n_local + kSTR - 1) / kSTR;
  T* gX = (T*)p.X;
  T* gAX = (T*)p.AX;
  T* gG = (T*)p.G;
  const T* gV = (const T*)p.V;
  const T* gAV = (const T*)p.AV;
  auto arr = [&](int st, int a) { return (T*)(stg + st * S::stage + a * S::arr); };
  auto issue = [&](int st, int64_t tile) {
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, p.n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&full[st], (apply_update ? 5u : 3u) * b);
    const int64_t off = row0 * KP;
    bulk_g2s(arr(st, 0), gX + off, b, &full[st]);
    bulk_g2s(arr(st, 1), gAX + off, b, &full[st]);
    if (apply_update) {
      bulk_g2s(arr(st, 2), gV + off, b, &full[st]);
      bulk_g2s(arr(st, 3), gAV + off, b, &full[st]);
    }
    bulk_g2s(arr(st, 4), gG + off, b, &full[st]);
  };
  constexpr int NCW = kThreads / 32;               // compute warps
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&adone[s], NCW);
      mbar_init(&cdone[s], NCW);
    }
    fence_barrier_init();
  }
  if (tid < KP) s_alpha[tid] = apply_update ? p.alpha[tid] : 0.0;
  __syncthreads();
  if (warp == NCW) {
    // ---- producer warp: loads, stores, stage recycling (lane 0)
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
        if (tile < ntiles) issue(s, tile);
      }
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % NS;
        const uint32_t ph = (uint32_t)((it / NS) & 1);
        const int64_t row0 = tile * kSTR;
        const int rows = (int)imin64(kSTR, p.n_local - row0);
        const uint32_t b = (uint32_t)rows * KP * sizeof(T);
        mbar_wait(&adone[st], ph);
        if (apply_update) {
          bulk_s2g(gX + row0 * KP, arr(st, 0), b);
          bulk_s2g(gAX + row0 * KP, arr(st, 1), b);
          bulk_commit();
        }
        mbar_wait(&cdone[st], ph);
        bulk_s2g(gG + row0 * KP, arr(st, 4), b);
        bulk_commit();
        const int64_t nxt = tile + (int64_t)NS * gridDim.x;
        if (nxt < ntiles) {
          bulk_wait_read_all();                 // stage st no longer read by the stores
          issue(st, nxt);
        }
      }
      bulk_wait_all();
    }
    return;
  }
  // ---- compute warps (k_update_direction's phases A, B, C)
  const bool mma_warp = warp < NB;
  const int cb = mma_warp ? warp : 0;
  double bm[KS], bw[F1 ? 1 : KS];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int j = 4 * kk + tig, c = cb * 8 + gid;
    const bool keep = !TRI || j <= c;
    bm[kk] = keep ? p.M[j * KP + c] : 0.0;
    if (!F1) bw[kk] = keep ? p.W[j * KP + c] : 0.0;
  }
  double gg[2] = {0.0, 0.0}, dg[2] = {0.0, 0.0};
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % NS;
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, p.n_local - row0);
    mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
    named_bar_sync(1, kThreads);                 // last tile's phase C done with Xp / AXp
    T* sX = arr(st, 0);
    T* sAX = arr(st, 1);
    const T* sV = arr(st, 2);
    const T* sAV = arr(st, 3);
    T* sG = arr(st, 4);
    for (int e = tid; e < kSTR * KP; e += kThreads) {
      const int r = e / KP, c = e % KP;
      double x = 0.0, ax = 0.0;
      if (r < rows) {
        x = (double)sX[e];
        ax = (double)sAX[e];
        if (apply_update) {
          x = rndT<T>(fma(s_alpha[c], (double)sV[e], x));
          ax = rndT<T>(fma(s_alpha[c], (double)sAV[e], ax));
          sX[e] = (T)x;
          sAX[e] = (T)ax;
        }
      }
      Xp[r * LD + c] = x;
      AXp[r * LD + c] = ax;
    }
    fence_proxy_async_smem();
    named_bar_sync(1, kThreads);
    if (lane == 0) mbar_arrive(&adone[st]);
    if (mma_warp) {
      double a1[2][2] = {{0, 0}, {0, 0}}, a2[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        if (TRI && 4 * kk > 8 * cb + 7) continue;
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int o = (rb * 8 + gid) * LD + 4 * kk + tig;
          const double xa = Xp[o];
          if (F1) {
            dmma(a1[rb][0], a1[rb][1], xa, bm[kk]);
          } else {
            const double aa = AXp[o];
            dmma(a1[rb][0], a1[rb][1], xa, bw[kk]);
            dmma(a2[rb][0], a2[rb][1], aa, bm[kk]);
          }
        }
      }
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) {
        const int r = rb * 8 + gid;
        if (r < rows) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = cb * 8 + 2 * tig + h;
            const double ax = AXp[r * LD + c];
            double g;
            // explicit roundings: every C3 variant computes the same bits
            if (METHOD == OFSC_OFM_F1) g = fma(4.0, a1[rb][h], 4.0 * ax);
            else if (METHOD == OFSC_TRIOFM_F1) g = __dadd_rn(ax, a1[rb][h]);
            else if (METHOD == OFSC_OFM_F2) g = fma(-2.0, a2[rb][h], fma(-2.0, a1[rb][h], 4.0 * ax));
            else g = __dadd_rn(__dadd_rn(2.0 * ax, -a2[rb][h]), -a1[rb][h]);
            g = rndT<T>(g);
            const double gp = (double)sG[r * KP + c];
            sG[r * KP + c] = (T)g;
            gg[h] = fma(g, g, gg[h]);
            dg[h] = fma(g - gp, g, dg[h]);
          }
        }
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&cdone[st]);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      gg[h] += __shfl_xor_sync(0xffffffffu, gg[h], o);
      dg[h] += __shfl_xor_sync(0xffffffffu, dg[h], o);
    }
  if (mma_warp && gid == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = cb * 8 + 2 * tig + h;
      p.part_cols[(int64_t)blockIdx.x * 2 * KP + c] = gg[h];
      p.part_cols[(int64_t)blockIdx.x * 2 * KP + KP + c] = dg[h];
    }
  }
}

template <typename T, int KP, int METHOD>
static void launch_c3_ws(const IterParams& p, int apply, int nblk, cudaStream_t s) {
  const size_t smem = C3WsSmem<T, KP, METHOD>::bytes;
  auto kern = k_update_direction_ws<T, KP, METHOD>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kC3WsThreads), smem, s, pdl_take(), p, apply);
}

// Default: the warp-specialised C3 for the f1 methods (one DMMA product per tile:
// 86-88 registers, no spills; c4 OFM-f1 C3 3.30 -> 3.17 ms, 98 % of the HBM copy
// peak), the single-role kernel for the f2 methods (two products: at the 9-warp
// kernel's 96-register cap they spill, c4 OFM-f2 3.99 -> 4.37 ms;
// profiles/r02/c3_ws_ab.jsonl).  OFSC_C3_WS = 0 / 1 forces either kernel.
static int c3_ws(int method) {
  const char* e = getenv("OFSC_C3_WS");
  if (e && *e) return atoi(e);
  return method == OFSC_OFM_F1 || method == OFSC_TRIOFM_F1;
}

// OFSC_C3_TR8=1: the 8-row x 4-stage form of the single-role C3 (same bits).  Measured
// (profiles/r02/c3_tr8_ab.jsonl): the c4 OFM-f2 kernel 4.11-4.16 -> 3.84-3.93 ms in the
// profiling pass, but graph-launched iterations within noise at c4 (14.25-14.30 vs
// 14.39-14.44 ms OFM-f2, 14.22-14.26 vs 14.00-14.08 TriOFM-f2) and 4 % slower at c5
// (KP = 48): not the default.
static int c3_tr8() {
  const char* e = getenv("OFSC_C3_TR8");
  return (e && e[0] == '1') ? 1 : 0;
}

template <typename T, int KP, int METHOD, int TR, int NS>
static void launch_c3_form(const IterParams& p, int apply, int nblk, cudaStream_t s) {
  const size_t smem = C3Smem<T, KP, METHOD, TR, NS>::bytes;
  auto kern = k_update_direction<T, KP, METHOD, TR, NS>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kThreads), smem, s, pdl_take(), p, apply);
}

template <typename T, int KP, int METHOD>
static void launch_c3(const IterParams& p, int apply, int nblk, cudaStream_t s) {
  if (c3_tr8()) launch_c3_form<T, KP, METHOD, 8, 4>(p, apply, nblk, s);
  else launch_c3_form<T, KP, METHOD, kSTR, kC3Stages>(p, apply, nblk, s);
}

static int stream_grid(int64_t n_rows, size_t smem_bytes) {
  // resident CTAs per SM allowed by shared memory (227 KB usable, ~1 KB reserved per CTA)
  int per_sm = (int)((232448) / (smem_bytes + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  const int64_t tiles = (n_rows + kSTR - 1) / kSTR;
  int64_t g = (int64_t)num_sms() * per_sm;
  if (tiles < g) g = tiles;
  return (int)(g < 1 ? 1 : g);
}

int c3_grid(ofsc_dtype dt, int KP, int method, int64_t n) {
  size_t b = 0;
  OFSC_DISPATCH_KP(KP, {
    const bool f2 = method == OFSC_OFM_F2 || method == OFSC_TRIOFM_F2;
    if (dt == OFSC_F64) b = f2 ? C3Smem<double, KPC, 2>::bytes : C3Smem<double, KPC, 0>::bytes;
    else b = f2 ? C3Smem<float, KPC, 2>::bytes : C3Smem<float, KPC, 0>::bytes;
  });
  // at most 2 resident CTAs per SM: at KP = 48 a third fits in shared memory but
  // measured slower (c5 OFM-f2 2.072 -> 2.017 ms, TriOFM-f2 2.132 -> 1.987 ms per
  // iteration with 2; profiles/r02/c3_grid_ab.jsonl).  OFSC_C3_CTAS overrides (A/B).
  const char* e = getenv("OFSC_C3_CTAS");
  const int per_sm = (e && *e) ? atoi(e) : 2;
  const int64_t tiles = std::max<int64_t>(1, (n + kSTR - 1) / kSTR);
  return (int)std::min<int64_t>(std::min<int64_t>((int64_t)num_sms() * per_sm, tiles),
                                stream_grid(n, b));
}

void launch_update_direction(ofsc_dtype dt, const IterParams& p, int apply_update, int nblk,
                             cudaStream_t s) {
  OFSC_DISPATCH_KP(p.KP, {
    if (c3_ws(p.method)) {
      if (dt == OFSC_F64) {
        switch (p.method) {
          case 0: launch_c3_ws<double, KPC, 0>(p, apply_update, nblk, s); break;
          case 1: launch_c3_ws<double, KPC, 1>(p, apply_update, nblk, s); break;
          case 2: launch_c3_ws<double, KPC, 2>(p, apply_update, nblk, s); break;
          default: launch_c3_ws<double, KPC, 3>(p, apply_update, nblk, s); break;
        }
      } else {
        switch (p.method) {
          case 0: launch_c3_ws<float, KPC, 0>(p, apply_update, nblk, s); break;
          case 1: launch_c3_ws<float, KPC, 1>(p, apply_update, nblk, s); break;
          case 2: launch_c3_ws<float, KPC, 2>(p, apply_update, nblk, s); break;
          default: launch_c3_ws<float, KPC, 3>(p, apply_update, nblk, s); break;
        }
      }
      return;
    }
    if (dt == OFSC_F64) {
      switch (p.method) {
        case 0: launch_c3<double, KPC, 0>(p, apply_update, nblk, s); break;
        case 1: launch_c3<double, KPC, 1>(p, apply_update, nblk, s); break;
        case 2: launch_c3<double, KPC, 2>(p, apply_update, nblk, s); break;
        default: launch_c3<double, KPC, 3>(p, apply_update, nblk, s); break;
      }
    } else {
      switch (p.method) {
        case 0: launch_c3<float, KPC, 0>(p, apply_update, nblk, s); break;
        case 1: launch_c3<float, KPC, 1>(p, apply_update, nblk, s); break;
        case 2: launch_c3<float, KPC, 2>(p, apply_update, nblk, s); break;
        default: launch_c3<float, KPC, 3>(p, apply_update, nblk, s); break;
      }
    }
  });
}

// ---------------------------------------------------------------------------
// C4
// ---------------------------------------------------------------------------
template <typename T, int KP>
struct C4Smem {
  static constexpr int LD = KP + 4;
  static constexpr size_t pad = (size_t)kSTR * LD * 8;
  static constexpr size_t arr = (size_t)kSTR * KP * sizeof(T);
  static constexpr size_t stage = 3 * arr;                           // G, Vp, X
  static constexpr size_t bytes = 2 * pad + kSST * stage + KP * 8 + kSST * 8;
};

template <typename T, int KP>
__global__ void __launch_bounds__(kThreads, 2) k_direction_gram(IterParams p) {
  using S = C4Smem<T, KP>;
  constexpr int LD = S::LD;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* Vd = (double*)smraw;
  double* Xd = Vd + kSTR * LD;
  unsigned char* stg = smraw + 2 * S::pad;
  double* s_beta = (double*)(stg + kSST * S::stage);
  uint64_t* bar = (uint64_t*)(s_beta + KP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (p.n_local + kSTR - 1) / kSTR;
  const T* gG = (const T*)p.G;
  T* gV = (T*)p.V;
  const T* gX = (const T*)p.X;
  auto arr = [&](int st, int a) { return (T*)(stg + st * S::stage + a * S::arr); };  // 0 G, 1 V, 2 X
  auto issue = [&](int st, int64_t tile) {
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, p.n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&bar[st], 3u * b);
    bulk_g2s(arr(st, 0), gG + row0 * KP, b, &bar[st]);
    bulk_g2s(arr(st, 1), gV + row0 * KP, b, &bar[st]);
    bulk_g2s(arr(st, 2), gX + row0 * KP, b, &bar[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < kSST; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  if (tid < KP) s_beta[tid] = p.beta[tid];
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kSST; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < ntiles) issue(s, tile);
    }
  typename GramSel<KP>::type acc;   // Q = V^T V symmetric: upper blocks only at KP = 64
  acc.zero();
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kSST;
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, p.n_local - row0);
    mbar_wait(&bar[st], (uint32_t)((it / kSST) & 1));
    const T* sG = arr(st, 0);
    T* sV = arr(st, 1);
    const T* sX = arr(st, 2);
    for (int e = tid; e < kSTR * KP; e += kThreads) {
      const int r = e / KP, c = e % KP;
      double v = 0.0, x = 0.0;
      if (r < rows) {
        v = rndT<T>(fma(s_beta[c], (double)sV[e], -(double)sG[e]));
        x = (double)sX[e];
        sV[e] = (T)v;
      }
      Vd[r * LD + c] = v;
      Xd[r * LD + c] = x;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(gV + row0 * KP, sV, (uint32_t)rows * KP * sizeof(T));
      bulk_commit();
    }
    acc.accumulate(Vd, Vd, Vd, Xd, (rows + 3) & ~3, warp, lane);   // Q = V^T V, P = V^T X
    __syncthreads();
    if (tid == 0) {
      const int64_t nxt = tile + (int64_t)kSST * gridDim.x;
      if (nxt < ntiles) {
        bulk_wait_read_all();
        issue(st, nxt);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
  acc.store(p.part_g4 + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
}

template <typename T, int KP>
static void launch_c4(const IterParams& p, int nblk, cudaStream_t s) {
  const size_t smem = C4Smem<T, KP>::bytes;
  auto kern = k_direction_gram<T, KP>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kThreads), smem, s, pdl_take(), p);
}

// C4, warp-specialised (KP = 48 by default, see c4_ws):
// warps 8-11 (producers) wait for each TMA stage (G, Vp, X), form
// V = -G + beta Vp in place (the stage is then stored back as V by one bulk
// copy) and into a padded fp64 tile together with X, and hand the tile over on
// an mbarrier; warps 0-7 run the DMMA Grams Q = V^T V (upper blocks) and
// P = V^T X on it.  Same products and summation order as k_direction_gram.
template <typename T, int KP>
struct C4SmemWS {
  static constexpr int LD = KP + 4;
  static constexpr size_t pad = (size_t)kSTR * LD * 8;
  static constexpr size_t arr = (size_t)kSTR * KP * sizeof(T);
  static constexpr size_t stage = 3 * arr;                            // G, Vp (-> V), X
  static constexpr size_t bytes =
      kGWS_NP * 2 * pad + kGWS_NS * stage + KP * 8 + (kGWS_NS + 2 * kGWS_NP) * 8;
};

template <typename T, int KP>
__global__ void __launch_bounds__(kGWS_THREADS, 1) k_direction_gram_ws(IterParams p) {
  using S = C4SmemWS<T, KP>;
  constexpr int LD = S::LD;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (p.ctl->stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* pads = (double*)smraw;                                       // [NP][2][kSTR][LD]
  unsigned char* stg = smraw + kGWS_NP * 2 * S::pad;
  double* s_beta = (double*)(stg + kGWS_NS * S::stage);
  uint64_t* full = (uint64_t*)(s_beta + KP);
  uint64_t* pfull = full + kGWS_NS;
  uint64_t* pempty = pfull + kGWS_NP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (p.n_local + kSTR - 1) / kSTR;
  const T* gG = (const T*)p.G;
  T* gV = (T*)p.V;
  const T* gX = (const T*)p.X;
  auto arr = [&](int st, int a) { return (T*)(stg + st * S::stage + a * S::arr); };  // 0 G, 1 V, 2 X
  auto pad = [&](int pb, int a) { return pads + ((size_t)pb * 2 + a) * kSTR * LD; };
  auto issue = [&](int st, int64_t tile) {
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, p.n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&full[st], 3u * b);
    bulk_g2s(arr(st, 0), gG + row0 * KP, b, &full[st]);
    bulk_g2s(arr(st, 1), gV + row0 * KP, b, &full[st]);
    bulk_g2s(arr(st, 2), gX + row0 * KP, b, &full[st]);
  };
  if (tid == 0) {
    for (int s0 = 0; s0 < kGWS_NS; ++s0) mbar_init(&full[s0], 1);
    for (int s0 = 0; s0 < kGWS_NP; ++s0) {
      mbar_init(&pfull[s0], 1);
      mbar_init(&pempty[s0], 8);                 // one arrival per consumer warp
    }
    fence_barrier_init();
  }
  if (tid < KP) s_beta[tid] = p.beta[tid];
  __syncthreads();
  if (warp >= 8) {
    // ---- producers: V = -G + beta Vp (stage, in place, and padded), X padded
    const int ptid = tid - 256;
    if (ptid == 0)
      for (int s0 = 0; s0 < kGWS_NS; ++s0) {
        const int64_t tile = blockIdx.x + (int64_t)s0 * gridDim.x;
        if (tile < ntiles) issue(s0, tile);
      }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % kGWS_NS, pb = it % kGWS_NP;
      const int64_t row0 = tile * kSTR;
      const int rows = (int)imin64(kSTR, p.n_local - row0);
      mbar_wait(&full[st], (uint32_t)((it / kGWS_NS) & 1));
      if (it >= kGWS_NP) mbar_wait(&pempty[pb], (uint32_t)(((it / kGWS_NP) - 1) & 1));
      double* Vd = pad(pb, 0);
      double* Xd = pad(pb, 1);
      const T* sG = arr(st, 0);
      T* sV = arr(st, 1);
      const T* sX = arr(st, 2);
      for (int e = ptid; e < kSTR * KP; e += 128) {
        const int r = e / KP, c = e % KP;
        double v = 0.0, x = 0.0;
        if (r < rows) {
          v = rndT<T>(fma(s_beta[c], (double)sV[e], -(double)sG[e]));
          x = (double)sX[e];
          sV[e] = (T)v;
        }
        Vd[r * LD + c] = v;
        Xd[r * LD + c] = x;
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);                  // stage st transformed, tile pb written
      if (ptid == 0) {
        mbar_arrive(&pfull[pb]);
        bulk_s2g(gV + row0 * KP, sV, (uint32_t)rows * KP * sizeof(T));
        bulk_commit();
        const int64_t nxt = tile + (int64_t)kGWS_NS * gridDim.x;
        if (nxt < ntiles) {
          bulk_wait_read_all();                  // the V store has read stage st
          issue(st, nxt);
        }
      }
    }
    if (ptid == 0) bulk_wait_all();
  } else {
    // ---- consumers: Q = V^T V (upper blocks), P = V^T X on DMMA
    typename GramSel<KP>::type acc;
    acc.zero();
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int pb = it % kGWS_NP;
      const int rows = (int)imin64(kSTR, p.n_local - tile * kSTR);
      mbar_wait(&pfull[pb], (uint32_t)((it / kGWS_NP) & 1));
      const double* Vd = pad(pb, 0);
      const double* Xd = pad(pb, 1);
      acc.accumulate(Vd, Vd, Vd, Xd, (rows + 3) & ~3, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&pempty[pb]);
    }
    acc.store(p.part_g4 + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
  }
}

// warp-specialised C4 where it measured faster: KP = 48 (c5: 0.526 -> 0.453 ms);
// at KP = 64 the one 384-thread CTA per SM hides less DMMA latency than two
// staging-copy CTAs (c4 2.40 -> 2.75, c6 0.479 -> 0.556 ms), KP = 32 neutral-worse.
// OFSC_C4_WS=0/1 forces either kernel.
static int c4_ws(int KP) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("OFSC_C4_WS");
    v = (e && *e) ? atoi(e) : -1;
  }
  return v >= 0 ? v : (KP == 48 ? 1 : 0);
}

template <typename T, int KP>
static void launch_c4_ws(const IterParams& p, int nblk, cudaStream_t s) {
  const size_t smem = C4SmemWS<T, KP>::bytes;
  auto kern = k_direction_gram_ws<T, KP>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kGWS_THREADS), smem, s, pdl_take(), p);
}

int c4_grid(ofsc_dtype dt, int KP, int64_t n) {
  size_t b = 0;
  OFSC_DISPATCH_KP(KP, {
    if (c4_ws(KPC)) b = dt == OFSC_F64 ? C4SmemWS<double, KPC>::bytes : C4SmemWS<float, KPC>::bytes;
    else b = dt == OFSC_F64 ? C4Smem<double, KPC>::bytes : C4Smem<float, KPC>::bytes;
  });
  return stream_grid(n, b);
}

void launch_direction_gram(ofsc_dtype dt, const IterParams& p, int nblk, cudaStream_t s) {
  OFSC_DISPATCH_KP(p.KP, {
    if (c4_ws(KPC)) {
      if (dt == OFSC_F64) launch_c4_ws<double, KPC>(p, nblk, s);
      else launch_c4_ws<float, KPC>(p, nblk, s);
    } else {
      if (dt == OFSC_F64) launch_c4<double, KPC>(p, nblk, s);
      else launch_c4<float, KPC>(p, nblk, s);
    }
  });
}

// ---------------------------------------------------------------------------
// C2b: streaming Gram pair over own rows, from the SpMM output Y
//   mode 0 (iteration): T = Z^T Y (warps 0-3), R' = X^T Y (warps 4-7)
//   mode 1 (refresh):   M = Z^T Z,             W  = Z^T Y
// ---------------------------------------------------------------------------
template <typename T, int KP>
struct GSmem {
  static constexpr int LD = KP + 4;
  static constexpr size_t pad = (size_t)kSTR * LD * 8;
  static constexpr size_t arr = (size_t)kSTR * KP * sizeof(T);
  static constexpr size_t stage = 3 * arr;                            // Z, X, Y
  static constexpr size_t bytes = 3 * pad + kSST * stage + kSST * 8;
};

template <typename T, int KP, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
k_gram_stream(int64_t n_local, const T* __restrict__ gZ, const T* __restrict__ gX,
              const T* __restrict__ gY, double* __restrict__ part, const int* stop) {
  using S = GSmem<T, KP>;
  constexpr int LD = S::LD;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* Zd = (double*)smraw;
  double* Xd = Zd + kSTR * LD;
  double* Yd = Xd + kSTR * LD;
  unsigned char* stg = smraw + 3 * S::pad;
  uint64_t* bar = (uint64_t*)(stg + kSST * S::stage);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n_local + kSTR - 1) / kSTR;
  auto arr = [&](int st, int a) { return (const T*)(stg + st * S::stage + a * S::arr); };
  auto issue = [&](int st, int64_t tile) {
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&bar[st], (MODE == 0 ? 3u : 2u) * b);
    bulk_g2s((void*)arr(st, 0), gZ + row0 * KP, b, &bar[st]);
    if (MODE == 0) bulk_g2s((void*)arr(st, 1), gX + row0 * KP, b, &bar[st]);
    bulk_g2s((void*)arr(st, 2), gY + row0 * KP, b, &bar[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < kSST; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kSST; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < ntiles) issue(s, tile);
    }
  typename GramSel<KP>::type acc;   // T (or M) symmetric: upper blocks only at KP = 64
  acc.zero();
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kSST;
    const int rows = (int)imin64(kSTR, n_local - tile * kSTR);
    mbar_wait(&bar[st], (uint32_t)((it / kSST) & 1));
    const T* sZ = arr(st, 0);
    const T* sX = arr(st, 1);
    const T* sY = arr(st, 2);
    for (int e = tid; e < kSTR * KP; e += kThreads) {
      const int r = e / KP, c = e % KP;
      const bool ok = r < rows;
      Zd[r * LD + c] = ok ? (double)sZ[e] : 0.0;
      if (MODE == 0) Xd[r * LD + c] = ok ? (double)sX[e] : 0.0;
      Yd[r * LD + c] = ok ? (double)sY[e] : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t nxt = tile + (int64_t)kSST * gridDim.x;
      if (nxt < ntiles) issue(st, nxt);            // stage st fully consumed above
    }
    const int r4 = (rows + 3) & ~3;
    if (MODE == 0) acc.accumulate(Zd, Yd, Xd, Yd, r4, warp, lane);
    else acc.accumulate(Zd, Zd, Zd, Yd, r4, warp, lane);
    __syncthreads();
  }
  acc.store(part + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
}

// C2b, warp-specialised: warps 0-7 run the DMMA Gram products, warps 8-11
// (producers) wait for each TMA stage, convert it into one of two padded fp64
// tiles and hand it over on an mbarrier, so the tensor-pipe warps never wait
// for the staging copy.  Same products and summation order as k_gram_stream.

template <typename T, int KP>
struct GSmemWS {
  static constexpr int LD = KP + 4;
  static constexpr size_t pad = (size_t)kSTR * LD * 8;               // one padded array
  static constexpr size_t arr = (size_t)kSTR * KP * sizeof(T);
  static constexpr size_t stage = 3 * arr;                            // Z, X, Y
  static constexpr size_t bytes = kGWS_NP * 3 * pad + kGWS_NS * stage + (kGWS_NS + 2 * kGWS_NP) * 8;
};

template <typename T, int KP, int MODE>
__global__ void __launch_bounds__(kGWS_THREADS, 1)
k_gram_stream_ws(int64_t n_local, const T* __restrict__ gZ, const T* __restrict__ gX,
                 const T* __restrict__ gY, double* __restrict__ part, const int* stop) {
  using S = GSmemWS<T, KP>;
  constexpr int LD = S::LD;
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* pads = (double*)smraw;                                       // [NP][3][kSTR][LD]
  unsigned char* stg = smraw + kGWS_NP * 3 * S::pad;
  uint64_t* full = (uint64_t*)(stg + kGWS_NS * S::stage);
  uint64_t* pfull = full + kGWS_NS;
  uint64_t* pempty = pfull + kGWS_NP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n_local + kSTR - 1) / kSTR;
  auto arr = [&](int st, int a) { return (const T*)(stg + st * S::stage + a * S::arr); };
  auto pad = [&](int pb, int a) { return pads + ((size_t)pb * 3 + a) * kSTR * LD; };
  auto issue = [&](int st, int64_t tile) {
    const int64_t row0 = tile * kSTR;
    const int rows = (int)imin64(kSTR, n_local - row0);
    const uint32_t b = (uint32_t)rows * KP * sizeof(T);
    mbar_arrive_expect_tx(&full[st], (MODE == 0 ? 3u : 2u) * b);
    bulk_g2s((void*)arr(st, 0), gZ + row0 * KP, b, &full[st]);
    if (MODE == 0) bulk_g2s((void*)arr(st, 1), gX + row0 * KP, b, &full[st]);
    bulk_g2s((void*)arr(st, 2), gY + row0 * KP, b, &full[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < kGWS_NS; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < kGWS_NP; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], 8);                 // one arrival per consumer warp
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp >= 8) {
    // ---- producers: TMA stage -> padded fp64 tile
    const int ptid = tid - 256;
    if (ptid == 0)
      for (int s = 0; s < kGWS_NS; ++s) {
        const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
        if (tile < ntiles) issue(s, tile);
      }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % kGWS_NS, pb = it % kGWS_NP;
      const int rows = (int)imin64(kSTR, n_local - tile * kSTR);
      mbar_wait(&full[st], (uint32_t)((it / kGWS_NS) & 1));
      if (it >= kGWS_NP) mbar_wait(&pempty[pb], (uint32_t)(((it / kGWS_NP) - 1) & 1));
      double* Zd = pad(pb, 0);
      double* Xd = pad(pb, 1);
      double* Yd = pad(pb, 2);
      const T* sZ = arr(st, 0);
      const T* sX = arr(st, 1);
      const T* sY = arr(st, 2);
      for (int e = ptid; e < kSTR * KP; e += 128) {
        const int r = e / KP, c = e % KP;
        const bool ok = r < rows;
        Zd[r * LD + c] = ok ? (double)sZ[e] : 0.0;
        if (MODE == 0) Xd[r * LD + c] = ok ? (double)sX[e] : 0.0;
        Yd[r * LD + c] = ok ? (double)sY[e] : 0.0;
      }
      named_bar_sync(1, 128);                  // stage st consumed, tile pb written
      if (ptid == 0) {
        mbar_arrive(&pfull[pb]);
        const int64_t nxt = tile + (int64_t)kGWS_NS * gridDim.x;
        if (nxt < ntiles) issue(st, nxt);
      }
    }
  } else {
    // ---- consumers: DMMA Gram products on the padded tiles
    typename GramSel<KP>::type acc;
    acc.zero();
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int pb = it % kGWS_NP;
      const int rows = (int)imin64(kSTR, n_local - tile * kSTR);
      mbar_wait(&pfull[pb], (uint32_t)((it / kGWS_NP) & 1));
      const double* Zd = pad(pb, 0);
      const double* Xd = pad(pb, 1);
      const double* Yd = pad(pb, 2);
      const int r4 = (rows + 3) & ~3;
      if (MODE == 0) acc.accumulate(Zd, Yd, Xd, Yd, r4, warp, lane);
      else acc.accumulate(Zd, Zd, Zd, Yd, r4, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&pempty[pb]);
    }
    acc.store(part + (int64_t)blockIdx.x * 2 * KP * KP, warp, lane);
  }
}

template <typename T, int KP, int MODE>
static void launch_gs_ws(int64_t n, const void* Z, const void* X, const void* Y, double* part,
                         const int* stop, int nblk, cudaStream_t st) {
  const size_t smem = GSmemWS<T, KP>::bytes;
  auto kern = k_gram_stream_ws<T, KP, MODE>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kGWS_THREADS), smem, st, pdl_take(), n, (const T*)Z,
           (const T*)X, (const T*)Y, part, stop);
}

static int gs_ws() {   // warp-specialised C2b (default; OFSC_GS_WS=0: staging-copy kernel)
  static int v = -1;     // measured: c4 2.30 -> 2.27 ms, c3 0.0987 -> 0.0952 ms
  if (v < 0) {
    const char* e = getenv("OFSC_GS_WS");
    v = (e && *e) ? atoi(e) : 1;
  }
  return v;
}

template <typename T, int KP, int MODE>
static void launch_gs(int64_t n, const void* Z, const void* X, const void* Y, double* part,
                      const int* stop, int nblk, cudaStream_t st) {
  const size_t smem = GSmem<T, KP>::bytes;
  auto kern = k_gram_stream<T, KP, MODE>;
  static bool set = false;
  if (!set) {
    OFSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  launch_k(kern, dim3(nblk), dim3(kThreads), smem, st, pdl_take(), n, (const T*)Z,
           (const T*)X, (const T*)Y, part, stop);
}

int gram_stream_grid(ofsc_dtype dt, int KP, int64_t n) {
  size_t b = 0;
  OFSC_DISPATCH_KP(KP, {
    if (gs_ws()) b = dt == OFSC_F64 ? GSmemWS<double, KPC>::bytes : GSmemWS<float, KPC>::bytes;
    else b = dt == OFSC_F64 ? GSmem<double, KPC>::bytes : GSmem<float, KPC>::bytes;
  });
  return stream_grid(n, b);
}

void launch_gram_stream(ofsc_dtype dt, int KP, int64_t n, const void* Zown, const void* Xown,
                        const void* Y, double* part, int mode, const int* stop, int nblk,
                        cudaStream_t st) {
  OFSC_DISPATCH_KP(KP, {
    if (gs_ws()) {
      if (dt == OFSC_F64) {
        if (mode == 0) launch_gs_ws<double, KPC, 0>(n, Zown, Xown, Y, part, stop, nblk, st);
        else launch_gs_ws<double, KPC, 1>(n, Zown, Xown, Y, part, stop, nblk, st);
      } else {
        if (mode == 0) launch_gs_ws<float, KPC, 0>(n, Zown, Xown, Y, part, stop, nblk, st);
        else launch_gs_ws<float, KPC, 1>(n, Zown, Xown, Y, part, stop, nblk, st);
      }
      return;
    }
    if (dt == OFSC_F64) {
      if (mode == 0) launch_gs<double, KPC, 0>(n, Zown, Xown, Y, part, stop, nblk, st);
      else launch_gs<double, KPC, 1>(n, Zown, Xown, Y, part, stop, nblk, st);
    } else {
      if (mode == 0) launch_gs<float, KPC, 0>(n, Zown, Xown, Y, part, stop, nblk, st);
      else launch_gs<float, KPC, 1>(n, Zown, Xown, Y, part, stop, nblk, st);
    }
  });
}

// ---------------------------------------------------------------------------
// C2b for the f1 methods: the diagonals of T = V^T AV and R' = X^T AV only.
// OFM-f1 and TriOFM-f1 read T and R' through tr T, tr R' (eq:f1-derivative,
// P:298-305) and T_ii, R'_ii (eq:alphai-f1) alone, and their directions
// (eq:gradientf1, eq:gradientg1) never read W = X^T A X, so the k x k products of
// the full Grams are not needed: this kernel streams V, X, AV once (3B, HBM-bound)
// and forms the 2k column dots sum_r V_rc AV_rc, sum_r X_rc AV_rc in fp64.
// A CTA owns a fixed contiguous row range; each thread owns two adjacent columns
// of every RPI-th row of it; warps' sums meet in shared memory in a fixed order,
// so the partials (part[blk][2][KP]) are deterministic for a given grid.
// ---------------------------------------------------------------------------
template <typename T, int KP>
__global__ void __launch_bounds__(256) k_gram_diag(int64_t n, int64_t rows_per_blk,
                                                   const T* __restrict__ Z,
                                                   const T* __restrict__ X,
                                                   const T* __restrict__ Y,
                                                   double* __restrict__ part,
                                                   const int* stop) {
  constexpr int LPR = KP / 2;               // lanes per row (two columns each)
  constexpr int RPI = 256 / LPR;            // rows per CTA step
  using V2 = typename Vec2<T>::type;
  __shared__ double red[RPI][2 * KP];
  pdl_wait();      // PDL: the predecessor kernel has completed (sm100.cuh)
  pdl_trigger();
  if (stop && *stop) return;
  const int sub = threadIdx.x / LPR, l = threadIdx.x % LPR;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t r1 = min(n, r0 + rows_per_blk);
  double t0 = 0, t1 = 0, q0 = 0, q1 = 0;
  if (sub < RPI) {
    int64_t r = r0 + sub;
    constexpr int U = 4;                    // rows in flight per thread
    for (; r + (U - 1) * RPI < r1; r += U * RPI) {
      V2 z[U], x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t o = (r + u * RPI) * KP + 2 * l;
        z[u] = __ldcs(reinterpret_cast<const V2*>(Z + o));
        x[u] = __ldcs(reinterpret_cast<const V2*>(X + o));
        y[u] = __ldcs(reinterpret_cast<const V2*>(Y + o));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        t0 = fma((double)z[u].x, (double)y[u].x, t0);
        t1 = fma((double)z[u].y, (double)y[u].y, t1);
        q0 = fma((double)x[u].x, (double)y[u].x, q0);
        q1 = fma((double)x[u].y, (double)y[u].y, q1);
      }
    }
    for (; r < r1; r += RPI) {
      const int64_t o = r * KP + 2 * l;
      const V2 z = __ldcs(reinterpret_cast<const V2*>(Z + o));
      const V2 x = __ldcs(reinterpret_cast<const V2*>(X + o));
      const V2 y = __ldcs(reinterpret_cast<const V2*>(Y + o));
      t0 = fma((double)z.x, (double)y.x, t0);
      t1 = fma((double)z.y, (double)y.y, t1);
      q0 = fma((double)x.x, (double)y.x, q0);
      q1 = fma((double)x.y, (double)y.y, q1);
    }
    red[sub][2 * l] = t0;
    red[sub][2 * l + 1] = t1;
    red[sub][KP + 2 * l] = q0;
    red[sub][KP + 2 * l + 1] = q1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * KP; c += blockDim.x) {
    double a = red[0][c];
#pragma unroll 4
    for (int s = 1; s < RPI; ++s) a += red[s][c];
    part[(int64_t)blockIdx.x * 2 * KP + c] = a;
  }
}

// two CTAs per SM (16 warps, 12 16-byte loads in flight per thread: enough to stream
// at HBM rate) and at least 64 rows per CTA; few partials for the fixed-order reduction
int gram_diag_grid(int64_t n) {
  const int64_t g = std::min<int64_t>((int64_t)num_sms() * 2, (n + 63) / 64);
  return (int)std::max<int64_t>(1, g);
}

void launch_gram_diag(ofsc_dtype dt, int KP, int64_t n, const void* Zown, const void* Xown,
                      const void* Y, double* part, const int* stop, int nblk, cudaStream_t st) {
  const int64_t per = (n + nblk - 1) / std::max(nblk, 1);
  OFSC_DISPATCH_KP(KP, {
    if (dt == OFSC_F64)
      launch_k(k_gram_diag<double, KPC>, dim3(nblk), dim3(256), 0, st, pdl_take(), n, per,
               (const double*)Zown, (const double*)Xown, (const double*)Y, part, stop);
    else
      launch_k(k_gram_diag<float, KPC>, dim3(nblk), dim3(256), 0, st, pdl_take(), n, per,
               (const float*)Zown, (const float*)Xown, (const float*)Y, part, stop);
  });
  OFSC_LAUNCH_CHECK();
}

}  // namespace ofsc

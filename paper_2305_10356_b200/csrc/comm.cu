// Collectives of the row-partitioned multi-GPU path:
// the halo exchange of V / X rows (grouped point-to-point) and the sums over
// ranks of the k x k Grams, column dots and K-means partials (P:456-460:
// "local product + Allreduce").
//
// Two transports behind one interface:
//  * NCCL (one process per GPU over NVLink / NVSwitch): grouped ncclSend/ncclRecv
//    for the halo; ncclAllGather of the per-rank partial buffers followed by a
//    fixed rank-order sum on the device, so every rank (and every run, whatever
//    algorithm NCCL picks) gets the same bits -- the deterministic cross-rank
//    reduction SURVEY 8(e) asks for, instead of ncclAllReduce.
//  * an in-process local world (ofsc_comm_create_local_world): p ranks on ONE
//    device, each driven by its own host thread.  A collective drains the
//    rank's stream, meets the other ranks at a host barrier, copies the peers'
//    posted device buffers with stream-ordered device-to-device copies, and
//    meets them again before any buffer is reused.  No kernel ever waits on
//    another rank's kernel (B200_PROFILING.md: such waits are not allowed on one
//    GPU); the arithmetic after the transport (the rank-order sum kernel, the
//    split SpMM) is the NCCL path's, so the emulation tests the p > 1 schedule
//    the multi-GPU run executes, bit for bit up to the transport.
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace ofsc {

struct LocalWorld {
  explicit LocalWorld(int n) : p(n), ptr(n, nullptr), off(n, nullptr) {}
  int p;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;        // per rank: the buffer it posted for this collective
  std::vector<const int64_t*> off;     // per rank: its per-peer send offsets (rows)
  bool broken = false;                 // a rank timed out: every later collective fails
  // Every rank must reach the barrier from its own host thread; a rank that never
  // arrives (a caller driving all ranks from one thread, or a rank that failed
  // outside a collective) would hang the others, so the wait is bounded
  // (OFSC_LOCAL_WORLD_TIMEOUT_S, default 600 s) and then fails with OFSC_ERR_STATE.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    OFSC_REQUIRE(!broken, OFSC_ERR_STATE, "local world broken by an earlier timed-out collective");
    const uint64_t g = gen;
    if (++arrived == p) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const char* e = getenv("OFSC_LOCAL_WORLD_TIMEOUT_S");
    const double limit = (e && *e) ? atof(e) : 600.0;
    if (!cv.wait_for(lk, std::chrono::duration<double>(limit),
                     [&] { return gen != g || broken; })) {
      broken = true;
      cv.notify_all();
      throw Error{OFSC_ERR_STATE, "local world: a rank did not reach a collective within "
                                  "OFSC_LOCAL_WORLD_TIMEOUT_S (each rank needs its own host "
                                  "thread and the same sequence of calls)"};
    }
    OFSC_REQUIRE(!broken, OFSC_ERR_STATE, "local world broken by a timed-out collective");
  }
};

std::shared_ptr<LocalWorld> make_local_world(int nranks) {
  return std::make_shared<LocalWorld>(nranks);
}

bool comm_active(const ofsc_comm_s* c) {
  return c && c->nranks > 1 && (c->nccl || c->world);
}

// out[i] = (((g_0[i] + g_1[i]) + g_2[i]) + ...) : rank order, identical on every rank
template <typename T>
__global__ void k_sum_ranks(const T* __restrict__ gather, int p, size_t count, T* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T acc = gather[i];
    for (int q = 1; q < p; ++q) acc += gather[(size_t)q * count + i];
    out[i] = acc;
  }
}

template <typename T>
static void comm_sum(ofsc_comm_s* c, T* buf, size_t count, T* gather, ncclDataType_t type,
                     cudaStream_t s) {
  if (!comm_active(c) || count == 0) return;
  const int p = c->nranks;
  if (c->nccl) {
    OFSC_NCCL(ncclAllGather(buf, gather, count, type, c->nccl, s));
  } else {
    LocalWorld& w = *c->world;
    OFSC_CUDA(cudaStreamSynchronize(s));          // this rank's partial is final
    w.ptr[c->rank] = buf;
    w.barrier();                                   // every rank's partial is final
    for (int q = 0; q < p; ++q)
      OFSC_CUDA(cudaMemcpyAsync(gather + (size_t)q * count, w.ptr[q], count * sizeof(T),
                                cudaMemcpyDeviceToDevice, s));
    OFSC_CUDA(cudaStreamSynchronize(s));
    w.barrier();                                   // nobody overwrites a partial still being read
  }
  const int blocks = (int)std::min<size_t>((count + 255) / 256, 1024);
  k_sum_ranks<T><<<blocks, 256, 0, s>>>(gather, p, count, buf);
  OFSC_LAUNCH_CHECK();
}

void comm_sum_f64(ofsc_comm_s* c, double* buf, size_t count, double* gather, cudaStream_t s) {
  comm_sum<double>(c, buf, count, gather, ncclFloat64, s);
}

void comm_sum_u64(ofsc_comm_s* c, unsigned long long* buf, size_t count,
                  unsigned long long* gather, cudaStream_t s) {
  comm_sum<unsigned long long>(c, buf, count, gather, ncclUint64, s);
}

void comm_exchange(ofsc_comm_s* c, ncclDataType_t type, size_t row_elems, size_t elem_bytes,
                   const void* sendbuf, const std::vector<int64_t>& send_cnt,
                   const std::vector<int64_t>& send_off, void* recvbuf,
                   const std::vector<int64_t>& recv_cnt, const std::vector<int64_t>& recv_off,
                   cudaStream_t s) {
  if (!comm_active(c)) return;
  const int p = c->nranks, r = c->rank;
  const size_t row_bytes = row_elems * elem_bytes;
  if (c->nccl) {
    OFSC_NCCL(ncclGroupStart());
    for (int q = 0; q < p; ++q) {
      if (q == r) continue;
      if (send_cnt[q] > 0)
        OFSC_NCCL(ncclSend((const char*)sendbuf + (size_t)send_off[q] * row_bytes,
                           (size_t)send_cnt[q] * row_elems, type, q, c->nccl, s));
      if (recv_cnt[q] > 0)
        OFSC_NCCL(ncclRecv((char*)recvbuf + (size_t)recv_off[q] * row_bytes,
                           (size_t)recv_cnt[q] * row_elems, type, q, c->nccl, s));
    }
    OFSC_NCCL(ncclGroupEnd());
    return;
  }
  LocalWorld& w = *c->world;
  OFSC_CUDA(cudaStreamSynchronize(s));             // packed rows are final
  w.ptr[r] = sendbuf;
  w.off[r] = send_off.data();
  w.barrier();
  for (int q = 0; q < p; ++q) {
    if (q == r || recv_cnt[q] == 0) continue;
    // peer q's rows for rank r start at q's send offset for r (the plan is symmetric:
    // q's send count to r equals r's receive count from q)
    OFSC_CUDA(cudaMemcpyAsync((char*)recvbuf + (size_t)recv_off[q] * row_bytes,
                              (const char*)w.ptr[q] + (size_t)w.off[q][r] * row_bytes,
                              (size_t)recv_cnt[q] * row_bytes, cudaMemcpyDeviceToDevice, s));
  }
  OFSC_CUDA(cudaStreamSynchronize(s));
  w.barrier();
}

}  // namespace ofsc

// Tensor-parallel exchange steps (§2.3: "two all-reduce operations per layer" of
// Megatron TP) for a LOCAL GROUP: `world` model handles on ONE device inside one process, each
// driven by its own host thread (SPMD, identical calls), standing in for one process per GPU.
//
// It exists so every world > 1 code path of run_hybrid_batch (column/row-parallel shards, bf16
// partials, the all-reduce-add fused into RMSNorm, the pending partial of the last layer, the
// vocab-parallel LM head + all-gather + permute) runs — and is parity-tested against the
// unsharded fp64 oracle — on a single GPU.  The product multi-GPU path uses NCCL (model.cu); the
// two share everything except these two collective primitives:
//
//   all-reduce (sum, bf16):  each rank publishes its partial, records an event, host barrier;
//     each rank's stream waits for every peer's event, then reduce_bf16_kernel writes
//     bf16(sum over ranks 0..world-1 in rank order, fp32 accumulate) into that rank's own result
//     buffer (every rank computes the identical result, as ncclAllReduce guarantees);
//     a second event + barrier + wait keeps any rank from overwriting its partial before every
//     peer has read it.
//   all-gather (fp32): the same protocol with peer-to-peer device copies.
//
// The barrier times out (a peer that failed never arrives) and reports ENCCL instead of hanging.
#include "common.cuh"
#include "model.hpp"

#include <algorithm>
#include <cstdlib>

#include <chrono>
#include <condition_variable>
#include <mutex>

namespace sarathi {

namespace {

constexpr int kMaxWorld = 8;

struct PeerPtrs {
  const __nv_bfloat16* p[kMaxWorld];
};

__global__ void reduce_bf16_kernel(PeerPtrs in, int world, __nv_bfloat16* __restrict__ out, size_t n8) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < world; ++r) {  // rank order: identical result on every rank
      const uint4 raw = *reinterpret_cast<const uint4*>(in.p[r] + i * 8);
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + i * 8) = o;
  }
}

}  // namespace

struct LocalGroup {
  int world = 0;
  int device = 0;
  int timeout_s = 120;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<const void*> slot;  // pointer each rank publishes for the current collective
  std::vector<int> joined;
  // fused all-reduce registry: rank r's partial double buffer and ready-flag array
  std::vector<__nv_bfloat16*> arbuf0, arbuf1;
  std::vector<unsigned int*> ready;

  // false on timeout / broken group (a peer failed and will never arrive)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return generation != gen || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

Status local_group_create(int world, int device, LocalGroup** out) {
  if (world < 2 || world > kMaxWorld) return Status::err(SARATHI_EINVAL, "local_group: world must be in [2, 8]");
  auto* g = new LocalGroup();
  g->world = world;
  g->device = device;
  if (const char* t = getenv("SARATHI_GROUP_TIMEOUT_S")) g->timeout_s = std::max(1, atoi(t));
  g->ev_ready.assign(world, nullptr);
  g->ev_done.assign(world, nullptr);
  g->slot.assign(world, nullptr);
  g->joined.assign(world, 0);
  g->arbuf0.assign(world, nullptr);
  g->arbuf1.assign(world, nullptr);
  g->ready.assign(world, nullptr);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (int r = 0; r < world; ++r) {
    if (cudaEventCreateWithFlags(&g->ev_ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_done[r], cudaEventDisableTiming) != cudaSuccess) {
      local_group_destroy(g);
      cudaSetDevice(prev);
      return Status::err(SARATHI_ECUDA, "local_group: event creation failed");
    }
  }
  cudaSetDevice(prev);
  *out = g;
  return Status::ok();
}

void local_group_destroy(LocalGroup* g) {
  if (!g) return;
  for (auto e : g->ev_ready)
    if (e) cudaEventDestroy(e);
  for (auto e : g->ev_done)
    if (e) cudaEventDestroy(e);
  delete g;
}

Status local_group_join(LocalGroup* g, int rank, int world, int device) {
  std::lock_guard<std::mutex> lk(g->mu);
  if (world != g->world || device != g->device)
    return Status::err(SARATHI_EINVAL, "init_model: local_group world/device mismatch");
  if (g->joined[rank]) return Status::err(SARATHI_EINVAL, "init_model: rank already joined the local group");
  g->joined[rank] = 1;
  return Status::ok();
}

void local_group_leave(LocalGroup* g, int rank) {
  std::lock_guard<std::mutex> lk(g->mu);
  g->joined[rank] = 0;
}

// Publish `mine`, barrier, order this rank's stream after every peer's `ready` event.
static Status exchange_begin(LocalGroup* g, int rank, const void* mine, cudaStream_t st) {
  g->slot[rank] = mine;
  if (cudaEventRecord(g->ev_ready[rank], st) != cudaSuccess) return Status::err(SARATHI_ECUDA, "group: event record");
  if (!g->barrier()) return Status::err(SARATHI_ENCCL, "local group: barrier timed out (a peer rank failed?)");
  for (int r = 0; r < g->world; ++r)
    if (r != rank && cudaStreamWaitEvent(st, g->ev_ready[r], 0) != cudaSuccess)
      return Status::err(SARATHI_ECUDA, "group: stream wait");
  return Status::ok();
}

// After this rank's reads of the peers' buffers: nobody may reuse its buffer until all have read.
static Status exchange_end(LocalGroup* g, int rank, cudaStream_t st) {
  if (cudaEventRecord(g->ev_done[rank], st) != cudaSuccess) return Status::err(SARATHI_ECUDA, "group: event record");
  if (!g->barrier()) return Status::err(SARATHI_ENCCL, "local group: barrier timed out (a peer rank failed?)");
  for (int r = 0; r < g->world; ++r)
    if (r != rank && cudaStreamWaitEvent(st, g->ev_done[r], 0) != cudaSuccess)
      return Status::err(SARATHI_ECUDA, "group: stream wait");
  return Status::ok();
}

void local_group_register(LocalGroup* g, int rank, __nv_bfloat16* const arbuf[2], unsigned int* ready) {
  std::lock_guard<std::mutex> lk(g->mu);
  g->arbuf0[rank] = arbuf[0];
  g->arbuf1[rank] = arbuf[1];
  g->ready[rank] = ready;
}

bool local_group_peers(LocalGroup* g, const __nv_bfloat16* peer_ar[2][8], unsigned int* peer_ready[8]) {
  std::lock_guard<std::mutex> lk(g->mu);
  for (int r = 0; r < g->world; ++r) {
    if (!g->arbuf0[r] || !g->ready[r]) return false;
    peer_ar[0][r] = g->arbuf0[r];
    peer_ar[1][r] = g->arbuf1[r];
    peer_ready[r] = g->ready[r];
  }
  return true;
}

Status local_fused_begin(LocalGroup* g, int rank, cudaStream_t st) { return exchange_begin(g, rank, nullptr, st); }
Status local_fused_end(LocalGroup* g, int rank, cudaStream_t st) { return exchange_end(g, rank, st); }

namespace {
struct FlagPtrs {
  unsigned int* f[8];
};
__global__ void signal_ready_kernel(FlagPtrs pf, int rank, int world, unsigned int epoch) {
  const int r = threadIdx.x;
  if (r < world) {
    __threadfence_system();  // the partial (written by the preceding GEMM) before the flag, system scope
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.f[r] + rank), "r"(epoch) : "memory");
  }
}
}  // namespace

cudaError_t launch_signal_ready(unsigned int* const peer_ready[8], int rank, int world, unsigned int epoch,
                                cudaStream_t st) {
  FlagPtrs pf{};
  for (int r = 0; r < world; ++r) pf.f[r] = peer_ready[r];
  signal_ready_kernel<<<1, 32, 0, st>>>(pf, rank, world, epoch);
  return cudaGetLastError();
}

Status local_allreduce_bf16(LocalGroup* g, int rank, const __nv_bfloat16* partial, __nv_bfloat16* result, size_t count,
                            int num_sms, cudaStream_t st) {
  if (count % 8) return Status::err(SARATHI_EINVAL, "local all-reduce: count % 8 != 0");
  Status s = exchange_begin(g, rank, partial, st);
  if (s.code != SARATHI_OK) return s;
  PeerPtrs pp{};
  for (int r = 0; r < g->world; ++r) pp.p[r] = static_cast<const __nv_bfloat16*>(g->slot[r]);
  const size_t n8 = count / 8;
  const int grid = static_cast<int>(std::min<size_t>((n8 + 255) / 256, static_cast<size_t>(4 * num_sms)));
  reduce_bf16_kernel<<<std::max(grid, 1), 256, 0, st>>>(pp, g->world, result, n8);
  if (cudaGetLastError() != cudaSuccess) return Status::err(SARATHI_ECUDA, "local all-reduce: launch");
  return exchange_end(g, rank, st);
}

Status local_allgather_f32(LocalGroup* g, int rank, const float* src, float* dst, size_t count, cudaStream_t st) {
  Status s = exchange_begin(g, rank, src, st);
  if (s.code != SARATHI_OK) return s;
  for (int r = 0; r < g->world; ++r)
    if (cudaMemcpyAsync(dst + static_cast<size_t>(r) * count, g->slot[r], count * sizeof(float), cudaMemcpyDeviceToDevice,
                        st) != cudaSuccess)
      return Status::err(SARATHI_ECUDA, "local all-gather: copy");
  return exchange_end(g, rank, st);
}

}  // namespace sarathi

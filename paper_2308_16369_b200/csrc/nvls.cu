// NVLink-SHARP (NVLS) variant of the fused TP all-reduce (§2.3: two
// all-reduces per layer on the critical path).  One process per GPU, NCCL 2.28 symmetric memory:
//   * the row-parallel GEMM's bf16 partial double buffer and the ready flags live in ONE
//     ncclMemAlloc'd buffer registered as a symmetric window (NCCL_WIN_COLL_SYMMETRIC);
//   * ncclDevCommCreate(lsaMultimem) gives a multicast (multimem) address for the window, so the
//     consuming RMSNorm reads the SUM over every rank's partial with one
//     multimem.ld_reduce.add.acc::f32 per 4 bf16 (the NVSwitch reduces in flight: T*H*2 bytes per
//     rank instead of the one-shot's (world-1)*T*H*2), and the ready flags are written to the peers
//     through their LSA (load/store-accessible) pointers;
//   * the pointers are plain virtual addresses, queried ONCE at init by a tiny kernel (the NCCL
//     device API is only needed there), then used by the same signal / consumer kernels as the
//     peer-memory fused path (model.cu allreduce()).
// Opt-in (SARATHI_TP_NVLS=1, world > 1 with NCCL); built and compiled (the consumer's SASS holds
// LDGMC), unmeasured: no multi-GPU box was available.
#include "model.hpp"

#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>

namespace sarathi {

namespace {

struct NvlsApi {
  bool ok = false;
  decltype(&ncclMemAlloc) memAlloc = nullptr;
  decltype(&ncclMemFree) memFree = nullptr;
  decltype(&ncclCommWindowRegister) winRegister = nullptr;
  decltype(&ncclCommWindowDeregister) winDeregister = nullptr;
  decltype(&ncclDevCommCreate) devCommCreate = nullptr;
  decltype(&ncclDevCommDestroy) devCommDestroy = nullptr;
};

NvlsApi* nvls_api() {
  static NvlsApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.memAlloc = reinterpret_cast<decltype(api.memAlloc)>(dlsym(h, "ncclMemAlloc"));
      api.memFree = reinterpret_cast<decltype(api.memFree)>(dlsym(h, "ncclMemFree"));
      api.winRegister = reinterpret_cast<decltype(api.winRegister)>(dlsym(h, "ncclCommWindowRegister"));
      api.winDeregister = reinterpret_cast<decltype(api.winDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
      api.devCommCreate = reinterpret_cast<decltype(api.devCommCreate)>(dlsym(h, "ncclDevCommCreate"));
      api.devCommDestroy = reinterpret_cast<decltype(api.devCommDestroy)>(dlsym(h, "ncclDevCommDestroy"));
      api.ok = api.memAlloc && api.memFree && api.winRegister && api.winDeregister && api.devCommCreate;
    }
  }
  return api.ok ? &api : nullptr;
}

// out[0..1] = multimem addresses of the two partial buffers, out[2 + r] = rank r's flag array
// (LSA pointer), out[2 + world + r] = rank r's partial buffer 0 (LSA pointer, for reference).
__global__ void nvls_query_kernel(ncclWindow_t win, ncclDevComm dc, size_t off0, size_t off1, size_t off_flags,
                                  int world, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  out[0] = reinterpret_cast<unsigned long long>(ncclGetLsaMultimemPointer(win, off0, dc));
  out[1] = reinterpret_cast<unsigned long long>(ncclGetLsaMultimemPointer(win, off1, dc));
  for (int r = 0; r < world; ++r) {
    out[2 + r] = reinterpret_cast<unsigned long long>(ncclGetLsaPointer(win, off_flags, r));
    out[2 + world + r] = reinterpret_cast<unsigned long long>(ncclGetLsaPointer(win, off0, r));
  }
}

}  // namespace

struct NvlsState {
  void* buf = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
};

Status nvls_setup(Model& m) {
  NvlsApi* api = nvls_api();
  if (!api) return Status::err(SARATHI_ENCCL, "NVLS all-reduce: NCCL >= 2.28 symmetric-memory API not found");
  if (!m.nccl) return Status::err(SARATHI_ENCCL, "NVLS all-reduce: NCCL communicator required");
  const size_t part = static_cast<size_t>(m.Tmax) * m.cfg.hidden * 2;
  const size_t off1 = (part + 4095) / 4096 * 4096, off_flags = 2 * off1;
  const size_t bytes = off_flags + 4096;
  auto* st = new NvlsState();
  m.nvls = st;
  ncclComm_t comm = static_cast<ncclComm_t>(m.nccl);
  if (api->memAlloc(&st->buf, bytes) != ncclSuccess) return Status::err(SARATHI_ENCCL, "ncclMemAlloc failed");
  if (cudaMemset(st->buf, 0, bytes) != cudaSuccess) return Status::err(SARATHI_ECUDA, "memset NVLS window");
  if (api->winRegister(comm, st->buf, bytes, &st->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess)
    return Status::err(SARATHI_ENCCL, "ncclCommWindowRegister failed");
  ncclDevCommRequirements req;
  std::memset(&req, 0, sizeof(req));
  req.lsaMultimem = true;
  if (api->devCommCreate(comm, &req, &st->dev) != ncclSuccess)
    return Status::err(SARATHI_ENCCL, "ncclDevCommCreate(lsaMultimem) failed (no NVLS on this system?)");
  st->dev_ok = true;
  unsigned long long* d_out = nullptr;
  if (cudaMalloc(&d_out, (2 + 2 * m.world) * sizeof(unsigned long long)) != cudaSuccess)
    return Status::err(SARATHI_ECUDA, "cudaMalloc");
  nvls_query_kernel<<<1, 32, 0, m.stream>>>(st->win, st->dev, 0, off1, off_flags, m.world, d_out);
  std::vector<unsigned long long> h(2 + 2 * m.world);
  const cudaError_t e = cudaMemcpyAsync(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost, m.stream);
  cudaStreamSynchronize(m.stream);
  cudaFree(d_out);
  if (e != cudaSuccess) return Status::err(SARATHI_ECUDA, "NVLS pointer query failed");
  char* base = static_cast<char*>(st->buf);
  m.arbuf[0] = reinterpret_cast<__nv_bfloat16*>(base);
  m.arbuf[1] = reinterpret_cast<__nv_bfloat16*>(base + off1);
  m.ready = reinterpret_cast<unsigned int*>(base + off_flags);
  m.mm_ar[0] = reinterpret_cast<const __nv_bfloat16*>(h[0]);
  m.mm_ar[1] = reinterpret_cast<const __nv_bfloat16*>(h[1]);
  for (int r = 0; r < m.world; ++r) {
    m.peer_ready[r] = reinterpret_cast<unsigned int*>(h[2 + r]);
    m.peer_ar[0][r] = reinterpret_cast<const __nv_bfloat16*>(h[2 + m.world + r]);
    m.peer_ar[1][r] = reinterpret_cast<const __nv_bfloat16*>(h[2 + m.world + r] + off1);
  }
  m.peers_ok = true;
  return Status::ok();
}

void nvls_teardown(Model& m) {
  auto* st = static_cast<NvlsState*>(m.nvls);
  if (!st) return;
  NvlsApi* api = nvls_api();
  ncclComm_t comm = static_cast<ncclComm_t>(m.nccl);
  if (api && comm) {
    if (st->dev_ok && api->devCommDestroy) api->devCommDestroy(comm, &st->dev);
    if (st->win) api->winDeregister(comm, st->win);
    if (st->buf) api->memFree(st->buf);
  }
  delete st;
  m.nvls = nullptr;
}

}  // namespace sarathi

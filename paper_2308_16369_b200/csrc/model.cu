// Engine behind the C ABI: model init (device-side weight generation), paged KV pools, and the
// per-iteration kernel sequence of one decode-maximal hybrid batch (§4.3).
//
// Per layer l (PAPER.md L193-203 block; TP per L249 §2.3):
//   a  = RMSNorm(h; g1)                           [rmsnorm kernel; + pending TP all-reduce]
//   q,K,V = a Wqkv^T, RoPE, KV append at slot[t]  [tcgen05 GEMM, EPI_QKV_ROPE]
//   o[0:p]  = prefill attention (chunk rows)      [prefill_attention]
//   o[p:T]  = decode attention (decode rows)      [decode_attention (+combine)]
//   h += o Wo^T                                   [GEMM EPI_ADD_F32 | TP: bf16 partial + ncclAllReduce]
//   b  = RMSNorm(h; g2)
//   f  = SiLU(b Wg^T) * (b Wu^T)                  [GEMM EPI_SILU_MUL | GELU: EPI_GELU]
//   h += f Wd^T                                   [GEMM EPI_ADD_F32 | TP: bf16 partial + ncclAllReduce]
// then logits = RMSNorm(h[rows]; g_f) Wlm^T for the R requested rows (vocab-parallel under TP).
#include "model.hpp"

#include <cstdio>
#include <cstdlib>

#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>

namespace sarathi {

namespace {

// debug (SARATHI_PREFILL_TRACE): the time a stream reaches this point
__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

// ---- NCCL, resolved at run time (only needed for world > 1) ----
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

NcclApi* nccl_api(std::string* err) {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
      api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.allGather && api.commDestroy;
    }
  }
  if (!api.ok) {
    if (err) *err = "NCCL unavailable (dlopen libnccl.so.2 failed; import torch first)";
    return nullptr;
  }
  return &api;
}

// Counter-based generator constants (synth/__init__.py spec).
constexpr int kWQ = 0, kWK = 1, kWV = 2, kWO = 3, kWG = 4, kWU = 5, kWD = 6, kG1 = 7, kG2 = 8;
constexpr int kEmbTau = 1 << 20, kGfTau = (1 << 20) + 1, kWlmTau = (1 << 20) + 2;
constexpr int kHostPerLayer = 9;  // host_tensors per layer: wq wk wv wo wg wu wd g1 g2 (= kWQ..kG2)

float weight_scale(double sigma) { return static_cast<float>(std::sqrt(3.0) * sigma / 16777216.0); }

}  // namespace

int nccl_unique_id(void* out128, std::string* err) {
  NcclApi* api = nccl_api(err);
  if (!api) return SARATHI_ENCCL;
  ncclUniqueId id;
  if (api->getUniqueId(&id) != ncclSuccess) {
    if (err) *err = "ncclGetUniqueId failed";
    return SARATHI_ENCCL;
  }
  std::memcpy(out128, &id, sizeof(id));
  return SARATHI_OK;
}

Status Model::check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return Status::ok();
  return Status::err(SARATHI_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
Status Model::dalloc(T** p, size_t count) {
  void* ptr = nullptr;
  cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return Status::err(SARATHI_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  allocations.push_back(ptr);
  *p = static_cast<T*>(ptr);
  return Status::ok();
}

Status Model::dalloc_padded(__nv_bfloat16** p, int rows, int cols) {
  const size_t n = static_cast<size_t>((rows + 127) / 128) * 128 * cols;
  Status s = dalloc(p, n);
  if (s.code != SARATHI_OK) return s;
  return check(cudaMemsetAsync(*p, 0, n * 2, stream), "memset weight padding");
}

#define SRET(x)                  \
  do {                           \
    Status _s = (x);             \
    if (_s.code != SARATHI_OK) return _s; \
  } while (0)

Status Model::init(const sarathi_model_config& c, const sarathi_dist& d, uint64_t seed_,
                   const void* const* host_tensors) {
  cfg = c;
  rank = d.rank;
  world = d.world;
  device = d.device;
  stream = static_cast<cudaStream_t>(d.stream);
  seed = seed_;
  const int H = c.hidden, hd = c.head_dim;
  if (c.n_layers < 1 || H < 64 || H % 64 || (hd != 64 && hd != 128) || c.n_heads < 1 || c.n_kv_heads < 1 ||
      c.n_heads % c.n_kv_heads || c.vocab < 1 || c.max_seq_len < 1 || c.max_tokens_per_batch < 1 ||
      c.max_tokens_per_batch > 8192 || (c.ffn_kind != SARATHI_FFN_SWIGLU && c.ffn_kind != SARATHI_FFN_GELU))
    return Status::err(SARATHI_EINVAL, "init_model: invalid model configuration");
  if (world < 1 || rank < 0 || rank >= world)
    return Status::err(SARATHI_EINVAL, "init_model: invalid rank/world");
  // pipeline stage (NEXT-4): contiguous layer range [l0, l0 + nl) of the L layers
  pp_stages = d.pp_stages > 0 ? d.pp_stages : 1;
  pp_stage = d.pp_stage;
  if (pp_stage < 0 || pp_stage >= pp_stages || pp_stages > c.n_layers)
    return Status::err(SARATHI_EINVAL, "init_model: need 0 <= pp_stage < pp_stages <= n_layers");
  l0 = static_cast<int>(static_cast<long long>(c.n_layers) * pp_stage / pp_stages);
  nl = static_cast<int>(static_cast<long long>(c.n_layers) * (pp_stage + 1) / pp_stages) - l0;
  if (c.n_heads % world || c.n_kv_heads % world || c.ffn_hidden % (64 * world) || c.vocab % world)
    return Status::err(SARATHI_EINVAL,
                       "init_model: n_heads, n_kv_heads, vocab must divide by world and ffn_hidden by 64*world");
  const int G = c.n_heads / c.n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return Status::err(SARATHI_EINVAL, "init_model: GQA group must be 1/2/4/8");
  nq_l = c.n_heads / world;
  nkv_l = c.n_kv_heads / world;
  q_dim_l = nq_l * hd;
  kv_dim_l = nkv_l * hd;
  qkv_rows = q_dim_l + 2 * kv_dim_l;
  h2_l = c.ffn_hidden / world;
  gu_rows = c.ffn_kind == SARATHI_FFN_SWIGLU ? 2 * h2_l : h2_l;
  vocab_l = c.vocab / world;
  if (q_dim_l % 64) return Status::err(SARATHI_EINVAL, "init_model: local q dim must be a multiple of 64");
  if (qkv_rows % 128 && hd == 128) return Status::err(SARATHI_EINVAL, "init_model: qkv rows not tile aligned");
  SRET(check(cudaSetDevice(device), "cudaSetDevice"));
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* pr = getenv("SARATHI_AUX_PRIORITY");  // experiment: "low" | "high" (default)
    SRET(check(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, pr && pr[0] == 'l' ? lo : hi), "aux stream"));
    SRET(check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event"));
    SRET(check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event"));
  }
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);

  if (world > 1 && d.local_group) {
    SRET(local_group_join(static_cast<LocalGroup*>(d.local_group), rank, world, device));
    group = static_cast<LocalGroup*>(d.local_group);
    if (!stream) {  // each rank of a local group needs its own stream
      SRET(check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "rank stream"));
      owns_stream = true;
    }
  } else if (world > 1) {
    std::string err;
    NcclApi* api = nccl_api(&err);
    if (!api) return Status::err(SARATHI_ENCCL, err);
    if (!d.nccl_unique_id) return Status::err(SARATHI_EINVAL, "init_model: nccl_unique_id required for world > 1");
    ncclUniqueId id;
    std::memcpy(&id, d.nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    ncclResult_t r = api->commInitRank(&comm, world, id, rank);
    if (r != ncclSuccess)
      return Status::err(SARATHI_ENCCL, std::string("ncclCommInitRank: ") + (api->errStr ? api->errStr(r) : "?"));
    nccl = comm;
  }

  // ---- weights, generated on device shard by shard ----
  const int L = c.n_layers;
  const double s_in = 1.0 / std::sqrt(static_cast<double>(H));
  const double depth = 1.0 / std::sqrt(2.0 * L);
  const double s_o = depth / std::sqrt(static_cast<double>(c.n_heads) * hd);
  const double s_d = depth / std::sqrt(static_cast<double>(c.ffn_hidden));
  std::vector<int> tau;
  std::vector<float> scl;
  std::vector<long long> base;
  int* d_tau = nullptr;
  float* d_scl = nullptr;
  long long* d_base = nullptr;
  const int max_rows = std::max({qkv_rows, gu_rows, H, vocab_l, c.vocab});
  SRET(dalloc(&d_tau, max_rows));
  SRET(dalloc(&d_scl, max_rows));
  SRET(dalloc(&d_base, max_rows));
  // host_tensors: logical (unsharded) bf16 tensors, nn.Linear [out, in] layout, indexed
  // [layer * kHostPerLayer + kind] (kind = kWQ..kG2) then emb, final gain, LM head
  const int n_host = L * kHostPerLayer + 3;
  auto host_ptr = [&](int t) -> const uint16_t* {  // generator tensor id -> host tensor
    int idx;
    if (t == kEmbTau) idx = L * kHostPerLayer;
    else if (t == kGfTau) idx = L * kHostPerLayer + 1;
    else if (t == kWlmTau) idx = L * kHostPerLayer + 2;
    else idx = (t / 16) * kHostPerLayer + t % 16;
    return idx < n_host ? static_cast<const uint16_t*>(host_tensors[idx]) : nullptr;
  };
  if (host_tensors) {
    for (int i = 0; i < n_host; ++i)
      if (!host_tensors[i] && !(c.ffn_kind == SARATHI_FFN_GELU && i < L * kHostPerLayer && i % kHostPerLayer == kWU))
        return Status::err(SARATHI_EINVAL, "init_model: host_tensors[" + std::to_string(i) + "] is NULL");
  }
  __nv_bfloat16* staging = nullptr;  // host path: row-major shard [rows][cols] before packing
  size_t staging_elems = 0;
  std::vector<uint16_t> hbuf;
  // host path: every packed row r is the contiguous segment [base[r], base[r] + cols) of logical
  // tensor tau[r] (shard_map), so the shard is gathered row by row, copied H2D and packed on device
  auto upload = [&](__nv_bfloat16* dst, int rows, int cols, int packed) -> Status {
    hbuf.resize(static_cast<size_t>(rows) * cols);
    for (int r = 0; r < rows; ++r)
      std::memcpy(hbuf.data() + static_cast<size_t>(r) * cols, host_ptr(tau[r]) + base[r], static_cast<size_t>(cols) * 2);
    // copies are ordered on the model stream: a pageable cudaMemcpy on the legacy stream may return
    // before its DMA lands, and a rank's non-blocking stream would not wait for it
    if (!packed) {
      SRET(check(cudaMemcpyAsync(dst, hbuf.data(), hbuf.size() * 2, cudaMemcpyHostToDevice, stream), "H2D weights"));
      return check(cudaStreamSynchronize(stream), "H2D sync");  // hbuf is reused
    }
    if (hbuf.size() > staging_elems) {
      if (staging) cudaFree(staging);
      staging = nullptr;
      SRET(check(cudaMalloc(&staging, hbuf.size() * 2), "cudaMalloc staging"));
      staging_elems = hbuf.size();
    }
    SRET(check(cudaMemcpyAsync(staging, hbuf.data(), hbuf.size() * 2, cudaMemcpyHostToDevice, stream), "H2D weights"));
    SRET(check(launch_pack_weight(staging, dst, rows, cols, stream), "pack weight"));
    ++launches;
    return check(cudaStreamSynchronize(stream), "pack sync");
  };
  struct StagingGuard {
    __nv_bfloat16** p;
    ~StagingGuard() { if (*p) cudaFree(*p); }
  } staging_guard{&staging};
  auto gen = [&](__nv_bfloat16* dst, int rows, int cols, int packed) -> Status {
    if (host_tensors) return upload(dst, rows, cols, packed);
    SRET(check(cudaMemcpyAsync(d_tau, tau.data(), rows * sizeof(int), cudaMemcpyHostToDevice, stream), "H2D"));
    SRET(check(cudaMemcpyAsync(d_scl, scl.data(), rows * sizeof(float), cudaMemcpyHostToDevice, stream), "H2D"));
    SRET(check(cudaMemcpyAsync(d_base, base.data(), rows * sizeof(long long), cudaMemcpyHostToDevice, stream), "H2D"));
    SRET(check(launch_weightgen(dst, rows, cols, d_tau, d_scl, d_base, seed, packed, stream), "weightgen"));
    ++launches;
    return check(cudaStreamSynchronize(stream), "weightgen sync");  // host vectors are reused
  };
  auto fill = [&](int rows) {
    tau.assign(rows, 0);
    scl.assign(rows, 0.f);
    base.assign(rows, 0);
  };
  layers.resize(nl);
  for (int l = l0; l < l0 + nl; ++l) {  // global layer index l (generator ids), local storage l - l0
    LayerWeights& w = layers[l - l0];
    // GEMM weights in the tile-major layout (rows padded to 128; padding zero)
    SRET(dalloc_padded(&w.qkv, qkv_rows, H));
    SRET(dalloc_padded(&w.o, H, q_dim_l));
    SRET(dalloc_padded(&w.gu, gu_rows, H));
    SRET(dalloc_padded(&w.down, H, h2_l));
    SRET(dalloc(&w.g1, H));
    SRET(dalloc(&w.g2, H));
    // rank-local shards of the logical weights (host_sched.cpp: shard_map), generated on device
    ShardDims sd;
    __nv_bfloat16* dsts[4] = {w.qkv, w.o, w.gu, w.down};
    for (int t = 0; t < 4; ++t) {
      shard_map(c.n_layers, H, c.n_heads, c.n_kv_heads, hd, c.ffn_hidden, c.vocab, c.ffn_kind, rank, world, l, t, &tau,
                &scl, &base, &sd);
      SRET(gen(dsts[t], sd.rows, sd.cols, 1));
    }
    if (!make_tmap_weight(&w.m_qkv, w.qkv, qkv_rows, H) || !make_tmap_weight(&w.m_o, w.o, H, q_dim_l) ||
        !make_tmap_weight(&w.m_gu, w.gu, gu_rows, H) || !make_tmap_weight(&w.m_down, w.down, H, h2_l))
      return Status::err(SARATHI_ECUDA, "cuTensorMapEncodeTiled failed for a weight");
    if (host_tensors) {
      SRET(check(cudaMemcpyAsync(w.g1, host_ptr(16 * l + kG1), H * 2, cudaMemcpyHostToDevice, stream), "H2D gain"));
      SRET(check(cudaMemcpyAsync(w.g2, host_ptr(16 * l + kG2), H * 2, cudaMemcpyHostToDevice, stream), "H2D gain"));
    } else {
      SRET(check(launch_gaingen(w.g1, H, 16 * l + kG1, 0, seed, stream), "gaingen"));
      SRET(check(launch_gaingen(w.g2, H, 16 * l + kG2, 0, seed, stream), "gaingen"));
      launches += 2;
    }
  }
  // embedding (replicated; first pipeline stage), final gain, LM head (vocab-parallel; last stage)
  if (pp_stage == 0) {
    SRET(dalloc(&emb, static_cast<size_t>(c.vocab) * H));
    ShardDims sd;
    shard_map(c.n_layers, H, c.n_heads, c.n_kv_heads, hd, c.ffn_hidden, c.vocab, c.ffn_kind, rank, world, 0, 16, &tau,
              &scl, &base, &sd);
    SRET(gen(emb, c.vocab, H, 0));
  }
  if (pp_stage == pp_stages - 1) {
  SRET(dalloc(&gf, H));
  if (host_tensors) {
    SRET(check(cudaMemcpyAsync(gf, host_ptr(kGfTau), H * 2, cudaMemcpyHostToDevice, stream), "H2D gain"));
  } else {
    SRET(check(launch_gaingen(gf, H, kGfTau, 0, seed, stream), "gaingen"));
    ++launches;
  }
  SRET(dalloc_padded(&lm, vocab_l, H));
  {
    ShardDims sd;
    shard_map(c.n_layers, H, c.n_heads, c.n_kv_heads, hd, c.ffn_hidden, c.vocab, c.ffn_kind, rank, world, 0, 18, &tau,
              &scl, &base, &sd);
  }
  SRET(gen(lm, vocab_l, H, 1));
  if (!make_tmap_weight(&m_lm, lm, vocab_l, H)) return Status::err(SARATHI_ECUDA, "tensor map (lm head)");
  }

  // RoPE tables (fp64 on host -> fp32), reading O-7
  {
    const int half = hd / 2;
    std::vector<float> th(static_cast<size_t>(half) * 2);
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(static_cast<double>(c.rope_base), -(2.0 * i) / hd);
      th[2 * i] = static_cast<float>(inv);
      th[2 * i + 1] = static_cast<float>(inv - static_cast<double>(th[2 * i]));
    }
    SRET(dalloc(&rope_theta, th.size()));
    SRET(check(cudaMemcpyAsync(rope_theta, th.data(), th.size() * 4, cudaMemcpyHostToDevice, stream), "H2D rope"));
    SRET(check(cudaStreamSynchronize(stream), "H2D rope sync"));  // th is a local
  }

  // activations / workspaces
  Tmax = c.max_tokens_per_batch;
  SRET(dalloc(&h, static_cast<size_t>(Tmax) * H));
  SRET(dalloc(&a, static_cast<size_t>(Tmax) * H));
  SRET(dalloc(&q, static_cast<size_t>(Tmax) * q_dim_l));
  if (!make_tmap_bf16(&m_q, q, static_cast<uint64_t>(Tmax), q_dim_l, q_dim_l, 128))
    return Status::err(SARATHI_ECUDA, "tensor map (q)");
  SRET(dalloc(&o, static_cast<size_t>(Tmax) * q_dim_l));
  SRET(dalloc(&f, static_cast<size_t>(Tmax) * h2_l));
  SRET(dalloc(&ar, static_cast<size_t>(Tmax) * H));
  if (group) SRET(dalloc(&ar_red, static_cast<size_t>(Tmax) * H));
  ar_res = ar;
  // fused all-reduce (NEXT-1): default in a local group (parity-tested on one GPU); for one process
  // per GPU it is opt-in (SARATHI_TP_FUSED=1: CUDA-IPC peer mappings, not yet measured on hardware)
  {
    const char* fe = getenv("SARATHI_TP_FUSED");
    tp_fused = world > 1 && (group ? !(fe && fe[0] == '0') : (fe && fe[0] == '1'));
    const char* nv = getenv("SARATHI_TP_NVLS");
    tp_nvls = world > 1 && !group && nv && nv[0] == '1';
  }
  if (tp_nvls) {
    tp_fused = true;
    SRET(nvls_setup(*this));
  } else if (tp_fused) {
    SRET(dalloc(&arbuf[0], static_cast<size_t>(Tmax) * H));
    SRET(dalloc(&arbuf[1], static_cast<size_t>(Tmax) * H));
    SRET(dalloc(&ready, 8));
    SRET(check(cudaMemsetAsync(ready, 0, 8 * sizeof(unsigned int), stream), "memset flags"));
    SRET(check(cudaStreamSynchronize(stream), "flags"));
    if (group) {
      local_group_register(group, rank, arbuf, ready);
    } else {
      SRET(ipc_exchange());
    }
  }
  SRET(dalloc(&af, static_cast<size_t>(Tmax) * H));
  SRET(dalloc(&logits_dev, static_cast<size_t>(Tmax) * c.vocab));
  if (world > 1) {
    SRET(dalloc(&logits_local, static_cast<size_t>(Tmax) * vocab_l));
    SRET(dalloc(&logits_gather, static_cast<size_t>(world) * Tmax * vocab_l));
  }
  gemm_ws_floats = static_cast<size_t>(96) << 20;  // lower half: slot partials; upper half: red.add partials
  SRET(dalloc(&gemm_ws, gemm_ws_floats));
  SRET(check(cudaMemset(gemm_ws + gemm_ws_floats / 2, 0, gemm_ws_floats / 2 * sizeof(float)), "zero ws"));
  SRET(dalloc(&gemm_counters, 1 << 16));
  SRET(check(cudaMemset(gemm_counters, 0, (1 << 16) * sizeof(int)), "memset"));
  part_cap = static_cast<size_t>(32) << 20;
  SRET(dalloc(&part_o, part_cap));
  SRET(dalloc(&part_lse, part_cap / 64 + 1024));
  pp_rows = static_cast<size_t>(64) << 10;  // 64 K rows of head_dim floats (32 MB at hd 128)
  SRET(dalloc(&pp_o, pp_rows * hd));
  SRET(dalloc(&pp_ml, 2 * pp_rows));
  pp_pairs = ((Tmax + 127) / 128) * nq_l;
  SRET(dalloc(&pp_ctr, pp_pairs));
  SRET(check(cudaMemset(pp_ctr, 0, pp_pairs * sizeof(int)), "memset"));
  SRET(dalloc(&norm_ctr, 1));
  SRET(check(cudaMemset(norm_ctr, 0, sizeof(unsigned)), "memset"));
  SRET(dalloc(&gemm_done, 1));
  SRET(check(cudaMemset(gemm_done, 0, sizeof(unsigned)), "memset"));
  SRET(dalloc(&norm_done, 1));
  SRET(check(cudaMemset(norm_done, 0, sizeof(unsigned)), "memset"));
  SRET(dalloc(&aflags, static_cast<size_t>(nkv_l + 1)));
  SRET(dalloc(&acnt, static_cast<size_t>(nkv_l + 1)));
  SRET(check(cudaMemset(aflags, 0, (nkv_l + 1) * sizeof(unsigned)), "memset"));
  SRET(check(cudaMemset(acnt, 0, (nkv_l + 1) * sizeof(int)), "memset"));
  // layer chain (world == 1; SARATHI_CHAIN=0 keeps one launch per GEMM + RMSNorm kernels)
  {
    const char* ce = getenv("SARATHI_CHAIN");
    // opt-in: measured no faster than the standalone PDL-chained GEMMs at [13B-1] (interleaved A/B,
    // profiles/r02_ab_drain.txt) and slower on TP-rank shapes; SARATHI_CHAIN=1 (policy: large-M
    // shapes) or 2 (every shape)
    chain_on = world == 1 && H % 128 == 0 && ce && (ce[0] == '1' || ce[0] == '2');
  }
  if (chain_on) {
    nt_h = 2 * ((H + 255) / 256);
    nt_gu = 2 * ((gu_rows + 255) / 256);
    SRET(dalloc(&a2, static_cast<size_t>(Tmax) * H));
    SRET(dalloc(&ss1, static_cast<size_t>(nt_h) * Tmax));
    SRET(dalloc(&ss2, static_cast<size_t>(nt_h) * Tmax));
    SRET(dalloc(&cflags, static_cast<size_t>(2 * nt_h + nt_gu)));
    nt_qkv = 2 * ((qkv_rows + 255) / 256);
    SRET(dalloc(&ccnt, static_cast<size_t>(2 * nt_h + 2 * nt_gu + 2 * nt_qkv)));
    // split-tile scratch of the whole-tile jobs (FFN1, QKV): one 256-column slab per pair tile
    scr_ld = (nt_gu + nt_qkv) * 128;
    SRET(dalloc(&cscr, static_cast<size_t>(Tmax) * scr_ld));
    SRET(check(cudaMemset(cscr, 0, static_cast<size_t>(Tmax) * scr_ld * sizeof(float)), "memset"));
    SRET(check(cudaMemset(cflags, 0, (2 * nt_h + nt_gu) * sizeof(unsigned)), "memset"));
    SRET(check(cudaMemset(ccnt, 0, (2 * nt_h + 2 * nt_gu + 2 * nt_qkv) * sizeof(int)), "memset"));
  }
  SRET(check(cudaStreamSynchronize(stream), "init sync"));
  return Status::ok();
}

// Multi-process fused all-reduce: every rank's partial double buffer and ready flags mapped into
// every other rank over CUDA IPC (handles exchanged with one ncclAllGather).
Status Model::ipc_exchange() {
  NcclApi* api = nccl_api(nullptr);
  if (!api || !nccl) return Status::err(SARATHI_ENCCL, "fused all-reduce: NCCL communicator required");
  constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
  std::vector<unsigned char> mine(3 * kH), all(static_cast<size_t>(world) * 3 * kH);
  void* ptrs[3] = {arbuf[0], arbuf[1], ready};
  for (int i = 0; i < 3; ++i) {
    cudaIpcMemHandle_t hd;
    SRET(check(cudaIpcGetMemHandle(&hd, ptrs[i]), "cudaIpcGetMemHandle"));
    std::memcpy(mine.data() + i * kH, &hd, kH);
  }
  unsigned char* dev = nullptr;
  SRET(dalloc(&dev, all.size()));
  SRET(check(cudaMemcpy(dev + static_cast<size_t>(rank) * 3 * kH, mine.data(), 3 * kH, cudaMemcpyHostToDevice), "H2D"));
  if (api->allGather(dev + static_cast<size_t>(rank) * 3 * kH, dev, 3 * kH, ncclUint8, static_cast<ncclComm_t>(nccl),
                     stream) != ncclSuccess)
    return Status::err(SARATHI_ENCCL, "ncclAllGather (IPC handles) failed");
  SRET(check(cudaStreamSynchronize(stream), "allgather sync"));
  SRET(check(cudaMemcpy(all.data(), dev, all.size(), cudaMemcpyDeviceToHost), "D2H"));
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      peer_ar[0][r] = arbuf[0];
      peer_ar[1][r] = arbuf[1];
      peer_ready[r] = ready;
      continue;
    }
    void* q[3];
    for (int i = 0; i < 3; ++i) {
      cudaIpcMemHandle_t hd;
      std::memcpy(&hd, all.data() + (static_cast<size_t>(r) * 3 + i) * kH, kH);
      SRET(check(cudaIpcOpenMemHandle(&q[i], hd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle"));
      ipc_opened.push_back(q[i]);
    }
    peer_ar[0][r] = static_cast<const __nv_bfloat16*>(q[0]);
    peer_ar[1][r] = static_cast<const __nv_bfloat16*>(q[1]);
    peer_ready[r] = static_cast<unsigned int*>(q[2]);
  }
  peers_ok = true;
  return Status::ok();
}

Status Model::alloc_kv(int64_t nb, int32_t bs) {
  if (kv_ready) return Status::err(SARATHI_ESTATE, "alloc_kv: already allocated");
  // block sizes the attention kernels tile: each divides the tcgen05 prefill kernel's 128-key tile,
  // and the decode kernel's smallest (2-stage) K/V ring, 2 x 2 x bs x hd x 2 B, fits shared memory
  if (nb < 1 || nb > (1ll << 31) - 1 || (bs != 16 && bs != 32 && bs != 64 && bs != 128))
    return Status::err(SARATHI_EINVAL, "alloc_kv: num_blocks >= 1 and block_size in {16, 32, 64, 128}");
  const size_t per = static_cast<size_t>(nb) * nkv_l * bs * cfg.head_dim;
  kpool.resize(nl);
  vpool.resize(nl);
  kmap.resize(nl);
  vmap.resize(nl);
  for (int l = 0; l < nl; ++l) {
    SRET(dalloc(&kpool[l], per));
    SRET(dalloc(&vpool[l], per));
    // zero once: slots never written (past a request's length inside a block, or in blocks a tile
    // rounds up to) are read by the attention kernels under a zero probability; they must be finite
    SRET(check(cudaMemsetAsync(kpool[l], 0, per * 2, stream), "memset kv"));
    SRET(check(cudaMemsetAsync(vpool[l], 0, per * 2, stream), "memset kv"));
    const long long rows = nb * static_cast<long long>(nkv_l) * bs;
    if (!make_tmap_kv(&kmap[l], kpool[l], rows, cfg.head_dim, bs) ||
        !make_tmap_kv(&vmap[l], vpool[l], rows, cfg.head_dim, bs))
      return Status::err(SARATHI_ECUDA, "alloc_kv: tensor map encode failed");
  }
  num_blocks = nb;
  block_size = bs;
  max_blocks_per_req = (cfg.max_seq_len + bs - 1) / bs;
  alloc = BlockAllocator(nb, bs);
  meta_ints = static_cast<size_t>(5) * Tmax + static_cast<size_t>(Tmax + 1) * max_blocks_per_req;
  SRET(dalloc(&meta_dev, meta_ints));
  for (int i = 0; i < 2; ++i) {
    void* hp = nullptr;
    SRET(check(cudaMallocHost(&hp, meta_ints * sizeof(int)), "cudaMallocHost"));
    meta_host_buf[i] = static_cast<int*>(hp);
    SRET(check(cudaEventCreateWithFlags(&meta_ev[i], cudaEventDisableTiming), "cudaEventCreate"));
  }
  kv_ready = true;
  return Status::ok();
}

Status Model::take_span(int op, unsigned long long** start, unsigned long long** end) {
  *start = *end = nullptr;
  if (!profiling) return Status::ok();
  if (!span_buf) {
    SRET(dalloc(&span_buf, 2 * kSpanCap));
    SRET(check(cudaMemsetAsync(span_buf, 0xFF, kSpanCap * 8, stream), "span init"));
    SRET(check(cudaMemsetAsync(span_buf + kSpanCap, 0, kSpanCap * 8, stream), "span init"));
  }
  if (static_cast<int>(span_ops.size()) < kSpanCap) {
    *start = span_buf + span_ops.size();
    *end = span_buf + kSpanCap + span_ops.size();
    span_ops.push_back(op);
  }
  return Status::ok();
}

Status Model::xmap(const void* X, int N, int K, int ldx, int box_rows, const CUtensorMap** out) {
  auto xk = std::make_tuple(X, N, K, box_rows);
  auto xi = xmaps.find(xk);
  if (xi == xmaps.end()) {
    CUtensorMap m;
    if (!make_tmap_bf16(&m, X, N, K, ldx, box_rows)) return Status::err(SARATHI_ECUDA, "tensor map (activation)");
    xi = xmaps.emplace(xk, m).first;
  }
  *out = &xi->second;
  return Status::ok();
}

// Schedule of the layer chain for T tokens (cached per (T, with_qkv)): host list schedule
// (host_sched.cpp schedule_chain) uploaded once; costs in k-block units, env
// SARATHI_CHAIN_COSTS="silu,qkv,add,fin" overrides them for experiments.
Status Model::chain_plan(int T, bool with_qkv, const ChainPlanDev** out) {
  auto key = std::make_pair(T, with_qkv ? 1 : 0);
  auto it = chain_plans.find(key);
  if (it != chain_plans.end()) {
    *out = &it->second;
    return Status::ok();
  }
  ChainPlanDev pd;
  if (!plan_chain_tiling(T, &pd.base)) return Status::err(SARATHI_EINVAL, "chain: T needs more than one token tile");
  static double costs[4] = {22.0, 27.0, 16.0, 6.0};
  static bool costs_read = false;
  if (!costs_read) {
    costs_read = true;
    if (const char* ce = getenv("SARATHI_CHAIN_COSTS"))
      sscanf(ce, "%lf,%lf,%lf,%lf", &costs[0], &costs[1], &costs[2], &costs[3]);
  }
  const int H = cfg.hidden;
  const bool swiglu = cfg.ffn_kind == SARATHI_FFN_SWIGLU;
  std::vector<ChainJobShape> jobs(with_qkv ? 4 : 3);
  jobs[0] = {(H + 255) / 256, q_dim_l / 64, true, -1, 0.0};
  jobs[1] = {(gu_rows + 255) / 256, H / 64, false, 1, swiglu ? costs[0] : costs[0]};
  jobs[2] = {(H + 255) / 256, h2_l / 64, true, swiglu ? 0 : 1, 0.0};
  if (with_qkv) jobs[3] = {(qkv_rows + 255) / 256, H / 64, false, 1, costs[1]};
  static const bool split_whole = getenv("SARATHI_CHAIN_SPLIT") && atoi(getenv("SARATHI_CHAIN_SPLIT")) == 1;
  pd.sch = schedule_chain(jobs, num_sms / 2, costs[2], costs[3], 4, split_whole);
  const ChainSchedule& sc = pd.sch;
  const int pairs = num_sms / 2;
  std::vector<int> blob(sc.segs);
  blob.insert(blob.end(), sc.seg_off.begin(), sc.seg_off.end());
  pd.need_gu = static_cast<int>(blob.size());
  blob.insert(blob.end(), sc.need[1].begin(), sc.need[1].end());
  pd.slab_gu = static_cast<int>(blob.size());
  for (int pt = 0; pt < jobs[1].pm_tiles; ++pt) blob.push_back(pt);
  if (with_qkv) {
    pd.need_qkv = static_cast<int>(blob.size());
    blob.insert(blob.end(), sc.need[3].begin(), sc.need[3].end());
    pd.slab_qkv = static_cast<int>(blob.size());
    for (int pt = 0; pt < jobs[3].pm_tiles; ++pt) blob.push_back(nt_gu / 2 + pt);
  }
  pd.need_o = static_cast<int>(blob.size());
  blob.insert(blob.end(), sc.need[0].begin(), sc.need[0].end());
  pd.need_f2 = static_cast<int>(blob.size());
  blob.insert(blob.end(), sc.need[2].begin(), sc.need[2].end());
  SRET(dalloc(&pd.dev, blob.size()));
  SRET(check(cudaMemcpy(pd.dev, blob.data(), blob.size() * sizeof(int), cudaMemcpyHostToDevice), "chain plan"));
  pd.base.segs = pd.dev;
  pd.base.seg_off = pd.dev + sc.segs.size();
  pd.base.pairs = pairs;
  pd.base.ss_ld = Tmax;
  if (getenv("SARATHI_CHAIN_PRINT")) {
    fprintf(stderr, "chain T=%d qkv=%d: %zu segments, predicted makespan %.1f k-blocks (job ends", T, with_qkv ? 1 : 0,
            sc.segs.size() / 4, sc.makespan);
    for (double e : sc.job_end) fprintf(stderr, " %.1f", e);
    fprintf(stderr, ")\n");
  }
  it = chain_plans.emplace(key, pd).first;
  *out = &it->second;
  return Status::ok();
}

// One layer's GEMM phase as a chain launch: O(l) + residual -> FFN1(l) -> FFN2(l) + residual ->
// [QKV(l+1) + RoPE + KV append] (see gemm_chain.cu).
Status Model::run_chain(int l, int T, bool with_qkv, const int* d_pos_dev, const int* d_slot_dev) {
  const ChainPlanDev* pd = nullptr;
  SRET(chain_plan(T, with_qkv, &pd));
  const int H = cfg.hidden;
  const bool swiglu = cfg.ffn_kind == SARATHI_FFN_SWIGLU;
  LayerWeights& w = layers[l];
  ChainLaunch cl = pd->base;
  ChainMaps maps;
  const int box = cl.bn / cl.n_mma / 2;
  unsigned* f_o = cflags;
  unsigned* f_gu = cflags + nt_h;
  unsigned* f_dn = cflags + nt_h + nt_gu;
  const CUtensorMap* mx = nullptr;
  cl.epoch = ++chain_epoch;
  if (cl.epoch == 0) cl.epoch = chain_epoch = 1;  // (2^32 launches) flags compare by signed difference
  cl.njobs = with_qkv ? 4 : 3;
  // job 0: O projection, h += o Wo^T; finalise: a2 = bf16(g2 * h), ss2
  {
    ChainJobDev& J = cl.job[0];
    J.ep.mode = EPI_ADD_F32;
    J.ep.out = h;
    J.ep.ldo = H;
    J.M = H;
    J.KB = q_dim_l / 64;
    J.fin_cnt = ccnt;
    J.fin_need = pd->dev + pd->need_o;
    J.fin_g = w.g2;
    J.fin_xa = a2;
    J.fin_ss = ss2;
    J.flag_out = f_o;
    maps.w[0] = w.m_o;
    SRET(xmap(o, T, q_dim_l, q_dim_l, box, &mx));
    maps.x[0] = *mx;
  }
  // job 1: FFN1 (gate||up + SiLU*up, or W1 + GELU) on a2, scaled by rsqrt(mean h^2 + eps)
  {
    ChainJobDev& J = cl.job[1];
    J.ep.mode = swiglu ? EPI_SILU_MUL : EPI_GELU;
    J.ep.out = f;
    J.ep.ldo = h2_l;
    J.M = gu_rows;
    J.KB = H / 64;
    J.dep_flag = f_o;
    J.dep_shift = 1;
    J.ss_in = ss2;
    J.ss_parts = H / 128;
    J.inv_h = 1.0f / static_cast<float>(H);
    J.eps = cfg.rms_eps;
    J.flag_out = f_gu;
    J.fin_need = pd->dev + pd->need_gu;  // split tiles reduce through scratch slabs
    J.slab = pd->dev + pd->slab_gu;
    J.arrive = ccnt + 2 * nt_h;
    J.written = ccnt + 2 * nt_h + nt_gu;
    maps.w[1] = w.m_gu;
    SRET(xmap(a2, T, H, H, box, &mx));
    maps.x[1] = *mx;
  }
  // job 2: FFN2, h += f Wd^T; finalise (when the next QKV follows): a = bf16(g1' * h), ss1
  {
    ChainJobDev& J = cl.job[2];
    J.ep.mode = EPI_ADD_F32;
    J.ep.out = h;
    J.ep.ldo = H;
    J.M = H;
    J.KB = h2_l / 64;
    J.dep_flag = f_gu;
    J.dep_shift = swiglu ? 0 : 1;
    if (with_qkv) {
      J.fin_cnt = ccnt + nt_h;
      J.fin_need = pd->dev + pd->need_f2;
      J.fin_g = layers[l + 1].g1;
      J.fin_xa = a;
      J.fin_ss = ss1;
      J.flag_out = f_dn;
    }
    maps.w[2] = w.m_down;
    SRET(xmap(f, T, h2_l, h2_l, box, &mx));
    maps.x[2] = *mx;
  }
  {
    // residual h [T][H] as the bulk reduce-add target (rows >= T clipped by the map)
    auto hk = std::make_tuple(static_cast<const void*>(h), T, H, -1);
    auto hi = xmaps.find(hk);
    if (hi == xmaps.end()) {
      CUtensorMap m;
      if (!make_tmap_f32_red(&m, h, T, H, H)) return Status::err(SARATHI_ECUDA, "tensor map (h reduce)");
      hi = xmaps.emplace(hk, m).first;
    }
    maps.hred = hi->second;
    auto sk = std::make_tuple(static_cast<const void*>(cscr), T, scr_ld, -1);
    auto si = xmaps.find(sk);
    if (si == xmaps.end()) {
      CUtensorMap m;
      if (!make_tmap_f32_red(&m, cscr, T, scr_ld, scr_ld)) return Status::err(SARATHI_ECUDA, "tensor map (scratch)");
      si = xmaps.emplace(sk, m).first;
    }
    maps.scr = si->second;
    cl.scr = cscr;
    cl.scr_ld = scr_ld;
  }
  if (with_qkv) {
    LayerWeights& wn = layers[l + 1];
    ChainJobDev& J = cl.job[3];
    EpiParams& e = J.ep;
    e.mode = EPI_QKV_ROPE;
    e.out = q;
    e.ldo = q_dim_l;
    e.pos = d_pos_dev;
    e.slot = d_slot_dev;
    e.rope_theta = rope_theta;
    e.kcache = kpool[l + 1];
    e.vcache = vpool[l + 1];
    e.head_dim = cfg.head_dim;
    e.n_q_local = nq_l;
    e.n_kv_local = nkv_l;
    e.block_size = block_size;
    J.M = qkv_rows;
    J.KB = H / 64;
    J.dep_flag = f_dn;
    J.dep_shift = 1;
    J.ss_in = ss1;
    J.ss_parts = H / 128;
    J.inv_h = 1.0f / static_cast<float>(H);
    J.eps = cfg.rms_eps;
    J.fin_need = pd->dev + pd->need_qkv;
    J.slab = pd->dev + pd->slab_qkv;
    J.arrive = ccnt + 2 * nt_h + 2 * nt_gu;
    J.written = ccnt + 2 * nt_h + 2 * nt_gu + nt_qkv;
    maps.w[3] = wn.m_qkv;
    SRET(xmap(a, T, H, H, box, &mx));
    maps.x[3] = *mx;
  }
  ++launches;
  SRET(take_span(SARATHI_OP_GEMM_CHAIN, &cl.span_start, &cl.span_end));
  // debug: SARATHI_CHAIN_TRACE=<T> prints the timeline of the first chain launch with T tokens
  // at layer 1 (per pair: segments with mainloop / epilogue stamps and producer dependency waits)
  static const char* ctr = getenv("SARATHI_CHAIN_TRACE");
  static bool ctraced = false;
  static unsigned long long* tr = nullptr;  // allocated and zeroed ahead so the traced launch keeps its PDL overlap
  const size_t n = static_cast<size_t>(cl.pairs) * kChainTraceSegs * 8 + 8;
  if (ctr && !tr) {
    cudaMalloc(&tr, n * 8);
    cudaMemset(tr, 0, n * 8);
    cudaDeviceSynchronize();
  }
  static int cmatch = 0;  // trace the 100th chain launch with T tokens (warm: a few steps in)
  if (ctr && !ctraced && atoi(ctr) == T && ++cmatch == 100) {
    ctraced = true;
    cl.trace = tr;
    const Status st = check(launch_chain(maps, cl, swiglu ? EPI_SILU_MUL : EPI_GELU, stream), "chain launch");
    std::vector<unsigned long long> hb(n);
    cudaStreamSynchronize(stream);
    cudaMemcpy(hb.data(), tr, n * 8, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = hb[static_cast<size_t>(cl.pairs) * kChainTraceSegs * 8];
    fprintf(stderr, "chain trace: grid dependency resolved at %.1f us after the first CTA started\n",
            (static_cast<double>(hb[static_cast<size_t>(cl.pairs) * kChainTraceSegs * 8 + 1]) - static_cast<double>(t0)) * 1e-3);
    auto us = [&](unsigned long long t) { return t ? (static_cast<double>(t) - static_cast<double>(t0)) * 1e-3 : -1.0; };
    double jmax[4][3] = {};  // per job: last commit, last published, sum of dep waits
    double jmin[4];
    for (double& x : jmin) x = 1e30;
    for (int c = 0; c < cl.pairs; ++c) {
      fprintf(stderr, "pair %2d:", c);
      for (int sgi = 0; sgi < kChainTraceSegs; ++sgi) {
        const unsigned long long* e = &hb[(static_cast<size_t>(c) * kChainTraceSegs + sgi) * 8];
        if (!e[0]) break;
        const int jb = static_cast<int>(e[6] >> 48), pt = static_cast<int>((e[6] >> 32) & 0xFFFF);
        const int k0 = static_cast<int>((e[6] >> 16) & 0xFFFF), k1 = static_cast<int>(e[6] & 0xFFFF);
        fprintf(stderr, " [j%d t%d %d-%d mma %.1f|%.1f-%.1f epi %.1f-%.1f-%.1f w%.1f]", jb, pt, k0, k1, us(e[0]), us(e[1]),
                us(e[2]), us(e[3]), us(e[7]), us(e[4]), e[5] * 1e-3);
        if (jb < 4) {
          jmin[jb] = std::min(jmin[jb], us(e[1]));
          jmax[jb][0] = std::max(jmax[jb][0], us(e[2]));
          jmax[jb][1] = std::max(jmax[jb][1], us(e[4]));
          jmax[jb][2] += e[5] * 1e-3;
        }
      }
      fprintf(stderr, "\n");
    }
    for (int jb = 0; jb < cl.njobs; ++jb)
      fprintf(stderr, "job %d: first stage %.1f us, last commit %.1f us, last published %.1f us, dep waits %.1f pair-us\n",
              jb, jmin[jb], jmax[jb][0], jmax[jb][1], jmax[jb][2]);
    return st;
  }
  return check(launch_chain(maps, cl, swiglu ? EPI_SILU_MUL : EPI_GELU, stream), "chain launch");
}

Status Model::gemm(const CUtensorMap& mw, int M, int K, const void* X, int ldx, int N, const EpiParams& ep_in, int op) {
  // SARATHI_DETERMINISTIC=1: no red.add reductions (bitwise run-to-run reproducible residual stream)
  static const bool deterministic = getenv("SARATHI_DETERMINISTIC") && atoi(getenv("SARATHI_DETERMINISTIC")) == 1;
  const bool atomic = ep_in.mode == EPI_ADD_F32;
  auto pk = std::make_tuple(M, N, K * 2 + (atomic ? 1 : 0));
  auto it = plans.find(pk);
  if (it == plans.end())
    it = plans.emplace(pk, plan_gemm(M, N, K, num_sms, gemm_ws_floats, 0, atomic, deterministic)).first;
  const GemmPlan& pl = it->second;
  const CUtensorMap *mx = nullptr, *mx2 = nullptr;
  SRET(xmap(X, N, K, ldx, pl.box_rows, &mx));
  SRET(xmap(X, N, K, ldx, pl.box_rows2, &mx2));
  EpiParams ep = ep_in;
  if (ep.done_ctr) gemm_done_arrivals += 2u * static_cast<unsigned>(pl.ctas);  // flag-chained RMSNorm
  if (ep.norm_h || ep.pnorm_out) {  // fused RMSNorm prologue / epilogue: grid barrier target = all arrivals so far + this grid
    norm_arrivals += 2u * static_cast<unsigned>(pl.ctas);
    ep.norm_ctr = norm_ctr;
    ep.norm_target = norm_arrivals;
  }
  ep.ws = gemm_ws;
  ep.ws_red = gemm_ws + gemm_ws_floats / 2;
  ep.counters = gemm_counters;
  ++launches;
  if (op >= 0) SRET(take_span(op, &ep.span_start, &ep.span_end));
  // debug: SARATHI_MODEL_TRACE=<epilogue mode>:<N> traces the first such launch with N tokens
  static const char* trace_env = getenv("SARATHI_MODEL_TRACE");
  static bool traced = false;
  const char* colon = trace_env ? strchr(trace_env, ':') : nullptr;
  if (colon && !traced && atoi(trace_env) == ep.mode && atoi(colon + 1) == N) {
    traced = true;
    unsigned long long* tr = nullptr;
    cudaMalloc(&tr, 4096 * 8);
    cudaMemsetAsync(tr, 0, 4096 * 8, stream);
    ep.trace = tr;
    if (const char* d = getenv("SARATHI_GEMM_DBG")) ep.dbg = atoi(d);  // traced launch only
    const Status st = check(launch_gemm(mw, *mx, *mx2, pl, ep, stream), "gemm launch");
    cudaStreamSynchronize(stream);
    dump_gemm_trace(tr, pl);
    cudaFree(tr);
    return st;
  }
  return check(launch_gemm(mw, *mx, *mx2, pl, ep, stream), "gemm launch");
}

cudaEvent_t Model::op_begin(cudaStream_t s) {
  // debug: SARATHI_SPANS_ONLY keeps the device spans but drops the per-op events, whose records
  // between kernels break the programmatic-dependent-launch chains (true launch gaps)
  static const bool spans_only = getenv("SARATHI_SPANS_ONLY") != nullptr;
  if (!profiling || spans_only) return nullptr;
  if (ev_used + 2 > ev_pool.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
  }
  cudaEvent_t b = ev_pool[ev_used++];
  cudaEventRecord(b, s ? s : stream);
  return b;
}

void Model::op_end(int op, cudaEvent_t b, cudaStream_t s) {
  if (!b) return;
  cudaEvent_t e = ev_pool[ev_used++];
  cudaEventRecord(e, s ? s : stream);
  pending_ops.emplace_back(op, b, e);
}

Status Model::collect_op_times() {
  SRET(check(cudaStreamSynchronize(stream), "op timers sync"));
  for (auto& t : pending_ops) {
    float ms = 0.f;
    SRET(check(cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t)), "cudaEventElapsedTime"));
    op_ms[std::get<0>(t)] += ms;
    op_count[std::get<0>(t)] += 1;
  }
  pending_ops.clear();
  ev_used = 0;
  if (!span_ops.empty()) {
    std::vector<unsigned long long> hs(2 * kSpanCap);
    SRET(check(cudaMemcpy(hs.data(), span_buf, hs.size() * 8, cudaMemcpyDeviceToHost), "span read"));
    for (size_t i = 0; i < span_ops.size(); ++i) {
      const unsigned long long a = hs[i], b = hs[kSpanCap + i];
      if (b > a) {
        op_kms[span_ops[i]] += (b - a) * 1e-6;
        op_kcount[span_ops[i]] += 1;
      }
    }
    static const int dump = getenv("SARATHI_SPAN_DUMP") ? atoi(getenv("SARATHI_SPAN_DUMP")) : 0;
    static bool dumped = false;
    if (dump > 0 && !dumped && !span_ops.empty()) {  // debug: timeline of the first `dump` spans
      dumped = true;
      const unsigned long long t0 = hs[0];
      unsigned long long prev_end = hs[kSpanCap];
      for (size_t i = 0; i < span_ops.size() && static_cast<int>(i) < dump; ++i)
        fprintf(stderr, "span op %2d: %9.3f .. %9.3f us (%7.3f us; gap from previous end %7.3f)\n", span_ops[i],
                (hs[i] - t0) * 1e-3, (hs[kSpanCap + i] - t0) * 1e-3, (hs[kSpanCap + i] - hs[i]) * 1e-3,
                i ? (static_cast<double>(hs[i]) - static_cast<double>(prev_end)) * 1e-3 : 0.0),
            prev_end = std::max(prev_end, hs[kSpanCap + i]);
    }
    span_ops.clear();
    SRET(check(cudaMemsetAsync(span_buf, 0xFF, kSpanCap * 8, stream), "span init"));
    SRET(check(cudaMemsetAsync(span_buf + kSpanCap, 0, kSpanCap * 8, stream), "span init"));
  }
  return Status::ok();
}

namespace {
// NVTX ranges (SURVEY §5 tracing): one per hybrid batch and one per layer, visible to nsys / ncu
// --nvtx; header-only nvtx3, a no-op when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

Status Model::run(const sarathi_prefill_chunk* pre, const sarathi_decode_set* dec, float* logits, int32_t flags) {
  NvtxRange nvtx_batch("sarathi_run_hybrid_batch");
  if (!kv_ready) return Status::err(SARATHI_ESTATE, "run_hybrid_batch: alloc_kv not called");
  // a pipeline stage before the last hands its residual stream on (sarathi_stage_output): no logits
  if (pp_stage != pp_stages - 1) flags = (flags | SARATHI_NO_LOGITS) & ~SARATHI_LOGITS_HOST;
  const int p = pre ? pre->n_tokens : 0;
  const int d = dec ? dec->n : 0;
  const int T = p + d;
  if (p < 0 || d < 0 || (pre && p == 0)) return Status::err(SARATHI_EINVAL, "run_hybrid_batch: empty chunk / negative count");
  if (T < 1 || T > Tmax) return Status::err(SARATHI_EINVAL, "run_hybrid_batch: T must be in [1, max_tokens_per_batch]");
  if (!logits && !(flags & SARATHI_NO_LOGITS)) return Status::err(SARATHI_EINVAL, "run_hybrid_batch: logits is NULL");
  // ---- validation (state unchanged on error) ----
  std::set<int64_t> seen;
  if (pre) {
    if (!pre->token_ids) return Status::err(SARATHI_EINVAL, "prefill token_ids NULL");
    if (!alloc.has(pre->req_id)) return Status::err(SARATHI_EUNKNOWN_REQ, "prefill request not allocated");
    if (pre->start_pos != cached.at(pre->req_id)) return Status::err(SARATHI_EPOS, "prefill start_pos != cached length");
    if (pre->start_pos + p > alloc.reserved(pre->req_id))
      return Status::err(SARATHI_EOVERFLOW, "prefill chunk exceeds the request's reservation");
    seen.insert(pre->req_id);
  }
  if (d > 0 && (!dec->req_ids || !dec->token_ids || !dec->positions))
    return Status::err(SARATHI_EINVAL, "decode arrays NULL");
  for (int j = 0; j < d; ++j) {
    const int64_t r = dec->req_ids[j];
    if (!alloc.has(r)) return Status::err(SARATHI_EUNKNOWN_REQ, "decode request not allocated");
    if (seen.count(r)) return Status::err(SARATHI_EDUP, "request appears twice in the batch");
    seen.insert(r);
    if (dec->positions[j] != cached.at(r) || dec->positions[j] < 1)
      return Status::err(SARATHI_EPOS, "decode position != cached length (or no prefix)");
    if (dec->positions[j] + 1 > alloc.reserved(r)) return Status::err(SARATHI_EOVERFLOW, "decode exceeds reservation");
  }
  for (int i = 0; i < p; ++i)
    if (pre->token_ids[i] < 0 || pre->token_ids[i] >= cfg.vocab) return Status::err(SARATHI_EINVAL, "token id out of range");
  for (int j = 0; j < d; ++j)
    if (dec->token_ids[j] < 0 || dec->token_ids[j] >= cfg.vocab) return Status::err(SARATHI_EINVAL, "token id out of range");
  if (pre && pre->start_pos + p > cfg.max_seq_len) return Status::err(SARATHI_EINVAL, "position >= max_seq_len");
  for (int j = 0; j < d; ++j)
    if (dec->positions[j] >= cfg.max_seq_len) return Status::err(SARATHI_EINVAL, "position >= max_seq_len");

  if (profiling && ev_used > 16384) SRET(collect_op_times());
  const bool all_rows = flags & SARATHI_RETURN_ALL_ROWS;
  const bool want_logits = !(flags & SARATHI_NO_LOGITS);
  const int R = all_rows ? T : d + (p > 0 ? 1 : 0);
  // ---- metadata (host, pinned) -> one H2D copy ----
  const size_t off_tok = 0, off_pos = Tmax, off_slot = 2 * static_cast<size_t>(Tmax), off_rows = 3 * static_cast<size_t>(Tmax),
               off_ctx = 4 * static_cast<size_t>(Tmax), off_ptab = 5 * static_cast<size_t>(Tmax),
               off_dtab = off_ptab + max_blocks_per_req;
  meta_flip ^= 1;
  int* mh = meta_host_buf[meta_flip];
  SRET(check(cudaEventSynchronize(meta_ev[meta_flip]), "metadata buffer reuse"));  // its last H2D finished
  last_slots.assign(T, 0);
  for (int i = 0; i < p; ++i) {
    const int pos = pre->start_pos + i;
    mh[off_tok + i] = pre->token_ids[i];
    mh[off_pos + i] = pos;
    mh[off_slot + i] = static_cast<int>(alloc.slot(pre->req_id, pos));
  }
  if (pre) {
    const auto& t = alloc.table(pre->req_id);
    for (int b = 0; b < max_blocks_per_req; ++b) mh[off_ptab + b] = b < static_cast<int>(t.size()) ? t[b] : 0;
  }
  for (int j = 0; j < d; ++j) {
    const int pos = dec->positions[j];
    mh[off_tok + p + j] = dec->token_ids[j];
    mh[off_pos + p + j] = pos;
    mh[off_slot + p + j] = static_cast<int>(alloc.slot(dec->req_ids[j], pos));
    mh[off_ctx + j] = pos + 1;
    const auto& t = alloc.table(dec->req_ids[j]);
    for (int b = 0; b < max_blocks_per_req; ++b)
      mh[off_dtab + static_cast<size_t>(j) * max_blocks_per_req + b] = b < static_cast<int>(t.size()) ? t[b] : 0;
  }
  for (int r = 0; r < R; ++r) mh[off_rows + r] = all_rows ? r : (p > 0 ? (r == 0 ? p - 1 : p + r - 1) : r);
  for (int i = 0; i < T; ++i) last_slots[i] = mh[off_slot + i];
  const size_t copy_ints = off_dtab + static_cast<size_t>(d) * max_blocks_per_req;
  SRET(check(cudaMemcpyAsync(meta_dev, mh, copy_ints * sizeof(int), cudaMemcpyHostToDevice, stream), "H2D metadata"));
  last_h2d = static_cast<int64_t>(copy_ints * sizeof(int));
  last_d2h = 0;
  SRET(check(cudaEventRecord(meta_ev[meta_flip], stream), "event record"));
  const int* d_tok = meta_dev + off_tok;
  const int* d_pos = meta_dev + off_pos;
  const int* d_slot = meta_dev + off_slot;
  const int* d_rows = meta_dev + off_rows;
  const int* d_ctx = meta_dev + off_ctx;
  const int* d_ptab = meta_dev + off_ptab;
  const int* d_dtab = meta_dev + off_dtab;

  const int H = cfg.hidden, hd = cfg.head_dim;
  const bool dump_layers = flags & SARATHI_DUMP_LAYERS;
  if (dump_layers && !dump) SRET(dalloc(&dump, static_cast<size_t>(nl + 1) * Tmax * H));
  if (pp_stage > 0 && !pp_in) return Status::err(SARATHI_ESTATE, "run_hybrid_batch: pipeline stage > 0 needs sarathi_stage_input");
  auto dump_h = [&](int idx) -> Status {
    if (!dump_layers) return Status::ok();
    return check(cudaMemcpyAsync(dump + static_cast<size_t>(idx) * Tmax * H, h, static_cast<size_t>(T) * H * 4,
                                 cudaMemcpyDeviceToDevice, stream),
                 "dump");
  };
  NcclApi* api = world > 1 && !group ? nccl_api(nullptr) : nullptr;
  if (tp_fused && !peers_ok) {
    if (!group || !local_group_peers(group, peer_ar, peer_ready))
      return Status::err(SARATHI_ESTATE, "fused all-reduce: not every rank of the group is initialised");
    peers_ok = true;
  }
  // TP all-reduce of a row-parallel GEMM's bf16 partial (2 per layer).  The GEMM
  // writes to ar_target(); allreduce() then leaves in `pend` what the consuming kernel (the next
  // RMSNorm, or the residual add) adds into h, and ar_end() runs after that consumer.
  //   NCCL: in-place ncclAllReduce, pend = the sum.  Local group, unfused: out-of-place summing
  //   kernel.  Fused (NEXT-1): signal the ranks' ready flags; pend = every rank's partial, summed
  //   by the consumer over peer memory (local group: + event/barrier ordering around it).
  PeerSum pend;
  bool pend_end = false;
  auto ar_target = [&]() -> __nv_bfloat16* { return tp_fused ? arbuf[ar_epoch & 1] : ar; };
  auto allreduce = [&]() -> Status {
    if (tp_fused) {
      const int b = static_cast<int>(ar_epoch & 1);
      ++ar_epoch;
      SRET(check(launch_signal_ready(peer_ready, rank, world, ar_epoch, stream), "signal"));
      ++launches;
      pend = PeerSum();
      pend.world = world;
      for (int r = 0; r < world; ++r) pend.p[r] = peer_ar[b][r];
      pend.ready = ready;
      pend.epoch = ar_epoch;
      pend.mm = tp_nvls ? mm_ar[b] : nullptr;
      if (group) {
        SRET(local_fused_begin(group, rank, stream));
        pend_end = true;
      }
      return Status::ok();
    }
    pend = PeerSum();
    pend.world = 1;
    if (group) {
      pend.p[0] = ar_red;
      ++launches;
      return local_allreduce_bf16(group, rank, ar, ar_red, static_cast<size_t>(T) * H, num_sms, stream);
    }
    pend.p[0] = ar;
    ncclResult_t r = api->allReduce(ar, ar, static_cast<size_t>(T) * H, ncclBfloat16, ncclSum,
                                    static_cast<ncclComm_t>(nccl), stream);
    if (r != ncclSuccess) return Status::err(SARATHI_ENCCL, "ncclAllReduce failed");
    return Status::ok();
  };
  auto ar_end = [&]() -> Status {  // after the consumer of `pend`
    if (!pend_end) return Status::ok();
    pend_end = false;
    return local_fused_end(group, rank, stream);
  };
  const PeerSum no_add;

  cudaEvent_t ob = op_begin();
  if (pp_stage == 0) {
    SRET(check(launch_embedding(d_tok, emb, h, T, H, stream), "embedding"));
  } else {  // pipeline: the previous stage's residual stream (fp32 [T][H], device)
    SRET(check(cudaMemcpyAsync(h, pp_in, static_cast<size_t>(T) * H * 4, cudaMemcpyDeviceToDevice, stream), "stage input"));
  }
  op_end(SARATHI_OP_EMBED, ob);
  ++launches;
  SRET(dump_h(0));
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  bool pending_ar = false;  // TP: down-proj partial in `ar` not yet added to h
  static const bool no_aux = getenv("SARATHI_NO_AUX") != nullptr;  // experiment: serial attention
  static const bool attn_chain = !(getenv("SARATHI_ATTN_CHAIN") && atoi(getenv("SARATHI_ATTN_CHAIN")) == 0);
  // layer chain: layer l's O -> FFN1 -> FFN2 and layer l+1's RMSNorm + QKV run as ONE launch
  // (gemm_chain.cu), so a layer after the first starts at its attention
  // (measured: a net gain only when the whole-tile jobs fill the GPU by themselves; a TP rank's
  // small-M QKV / FFN1 leave most pairs idle in the chain and run faster as standalone stream-K
  // GEMMs, profiles/r02_chain_*.txt; SARATHI_CHAIN=2 forces the chain for every shape)
  static const bool chain_force = getenv("SARATHI_CHAIN") && atoi(getenv("SARATHI_CHAIN")) == 2;
  const int pairs_avail = num_sms / 2;
  const bool chain_fits = 4 * ((gu_rows + 255) / 256) >= 3 * pairs_avail && 4 * ((qkv_rows + 255) / 256) >= 3 * pairs_avail;
  const bool use_chain = chain_on && gemm_token_tiling(T).n_tiles == 1 && (chain_fits || chain_force);
  // SARATHI_NORM_FUSED=1: RMSNorm fused into the next GEMM as a prologue + grid barrier (no
  // RMSNorm launch; world 1: no pending TP partial to add).  Measured slower than the PDL-chained
  // rmsnorm kernel (18.63 vs 18.51 ms, interleaved A/B, profiles/r02_ab_norm.txt): every CTA waits
  // for the slowest one before its first X load, so off by default.
  static const bool norm_fused_env = getenv("SARATHI_NORM_FUSED") && atoi(getenv("SARATHI_NORM_FUSED")) == 1;
  const bool norm_fused = norm_fused_env && world == 1;
  // SARATHI_POST_NORM=1: RMSNorm as the residual-add GEMM's epilogue (O -> norm2, down -> the next
  // layer's norm1; grid barrier + every CTA normalising rows): no rmsnorm launch and no
  // grid-completion gap before it (world 1, standalone GEMMs).  Parity-tested; measured slower than
  // the PDL-chained rmsnorm kernel (18.90 vs 18.80 ms interleaved A/B: O + norm 41-44 us vs 33 us,
  // the barrier waits for the slowest CTA's red.adds; profiles/r02_ab_pnorm.txt), so off by default.
  static const bool post_norm_env = getenv("SARATHI_POST_NORM") && atoi(getenv("SARATHI_POST_NORM")) == 1;
  const bool post_norm = post_norm_env && world == 1 && !norm_fused && !use_chain;
  bool normed_next = false;  // the previous layer's down GEMM already wrote this layer's norm1 into `a`
  // Flag-chained RMSNorm (world 1, standalone GEMMs): the residual-add GEMM's CTAs count themselves
  // in after their red.adds, the rmsnorm kernel waits on that count instead of the GEMM grid's
  // completion, and the next GEMM's TMA producer waits on the rmsnorm CTAs' count instead of the
  // rmsnorm grid's completion: the two grid-completion + launch gaps around every RMSNorm go.
  // Opt-in (SARATHI_NORM_FLAGS=1): parity-tested, measured slower (18.52 vs 18.06 ms interleaved
  // A/B: the early-resident rmsnorm CTAs stretch the norm to 5.9 us and gate||up by 11 us;
  // profiles/r02_ab_nflags.txt).
  static const bool norm_flags_env = getenv("SARATHI_NORM_FLAGS") && atoi(getenv("SARATHI_NORM_FLAGS")) == 1;
  const bool norm_flags = norm_flags_env && world == 1 && !norm_fused && !post_norm && !use_chain;
  bool flag_next = false;  // the previous layer's down GEMM counts into gemm_done (this layer's norm1 waits)
  auto flag_norm = [&](NormFlags& nf) {  // rmsnorm after a counting GEMM; returns via nf
    nf.wait_ctr = gemm_done;
    nf.wait_target = gemm_done_arrivals;
    nf.done_ctr = norm_done;
    norm_done_arrivals += static_cast<unsigned>(T);  // one CTA per row
  };
  auto flag_x = [&](EpiParams& e) {  // the GEMM after a flagged rmsnorm: X ready when all its CTAs counted in
    e.xflag = norm_done;
    e.xflag_cols = H;
    e.xflag_n = 1;
    e.xflag2 = nullptr;
    e.xepoch = norm_done_arrivals;
  };
  auto set_pnorm = [&](EpiParams& e, const __nv_bfloat16* g) {
    e.pnorm_g = g;
    e.pnorm_out = a;
    e.norm_T = T;
    e.norm_H = H;
    e.norm_eps = cfg.rms_eps;
  };
  auto set_norm = [&](EpiParams& e, const __nv_bfloat16* g) {
    e.norm_h = h;
    e.norm_g = g;
    e.norm_out = a;
    e.norm_T = T;
    e.norm_H = H;
    e.norm_eps = cfg.rms_eps;
  };
  for (int l = 0; l < nl; ++l) {  // this stage's layers (local index)
    NvtxRange nvtx_layer("layer");
    LayerWeights& w = layers[l];
    const bool flag1 = flag_next;
    flag_next = false;
    if ((l == 0 || !use_chain) && !norm_fused && !normed_next) {
    ob = op_begin();
    {
      unsigned long long *sp0, *sp1;
      SRET(take_span(SARATHI_OP_RMSNORM, &sp0, &sp1));
      NormFlags nf;
      if (flag1) flag_norm(nf);
      SRET(check(launch_rmsnorm(h, pending_ar ? pend : no_add, w.g1, a, nullptr, T, H, cfg.rms_eps, stream, sp0, sp1, nf),
                 "rmsnorm1"));
    }
    if (pending_ar) SRET(ar_end());
    op_end(SARATHI_OP_RMSNORM, ob);
    ++launches;
    pending_ar = false;
    }
    if (l > 0) SRET(dump_h(l));  // h after layer l-1 (TP: once the all-reduce has been added)
    if (l == 0 || !use_chain) {
    EpiParams e;
    if (norm_fused) set_norm(e, w.g1);
    if (flag1) flag_x(e);
    e.mode = EPI_QKV_ROPE;
    e.out = q;
    e.ldo = q_dim_l;
    e.pos = d_pos;
    e.slot = d_slot;
    e.rope_theta = rope_theta;
    e.kcache = kpool[l];
    e.vcache = vpool[l];
    e.head_dim = hd;
    e.n_q_local = nq_l;
    e.n_kv_local = nkv_l;
    e.block_size = block_size;
    ob = op_begin();
    SRET(gemm(w.m_qkv, qkv_rows, H, a, H, T, e, SARATHI_OP_GEMM_QKV));
    op_end(SARATHI_OP_GEMM_QKV, ob);
    }
    const bool chain = attn_chain && p > 0 && d > 0 && !no_aux;
    // SARATHI_O_EARLY=1: the O projection starts on finished KV heads inside the decode attention's
    // last wave (per-head flags instead of the grid dependency).  Measured: no earlier O completion
    // (the third split-K contributors need the last heads) and the decode slows by the overlap,
    // 18.79 vs 18.66 ms (profiles/r02_ab_oearly.txt), so off by default
    static const bool o_early = getenv("SARATHI_O_EARLY") && atoi(getenv("SARATHI_O_EARLY")) == 1;
    const bool xflags_try = o_early && d > 0 && (p == 0 || chain);
    bool xflags = false;
    if (xflags_try) ++attn_epoch;
    if (p > 0) {
      PrefillAttnArgs pa;
      pa.q = q;
      pa.q_ld = q_dim_l;
      pa.q_row0 = 0;
      pa.kcache = kpool[l];
      pa.vcache = vpool[l];
      pa.block_table = d_ptab;
      pa.start = pre->start_pos;
      pa.p = p;
      pa.n_q_local = nq_l;
      pa.n_kv_local = nkv_l;
      pa.head_dim = hd;
      pa.block_size = block_size;
      pa.scale = scale;
      pa.out = o;
      pa.out_ld = q_dim_l;
      pa.pdl = chain;
      {
        // key split for few (q-tile, head) pairs: when the chunk's attention (≈ 2.1 µs per
        // 128-key tile per CTA, the measured per-tile chain) would outlast the decode attention
        // beside it (its wave cost model below), or has the GPU to itself, its key tiles are
        // divided over up to 4 CTAs per pair (merged by the last; no range may be empty)
        const int ntq = (p + 127) / 128, pairs = ntq * nq_l;
        const int first_tiles = (pre->start_pos + std::min(128, p) + 127) / 128;
        const double est_p = 2.1 * ((pre->start_pos + p + 127) / 128);
        double est_d = 0.0;
        if (d > 0) {
          int mb = 0;
          for (int j = 0; j < d; ++j) mb = std::max(mb, (dec->positions[j] + 1 + block_size - 1) / block_size);
          const long long ctas = static_cast<long long>(d) * nkv_l;
          est_d = 1e30;
          for (int sp = 1; sp <= mb; ++sp) {
            const int bps = (mb + sp - 1) / sp;
            const double waves = static_cast<double>((ctas * sp + 2 * num_sms - 1) / (2 * num_sms));
            est_d = std::min(est_d, waves * (2.0 + 1.5 * bps) + (sp > 1 ? 3.0 : 0.0));
          }
        }
        int ks = 1;
        if (d > 0 ? est_p > 1.5 * est_d : 2 * pairs <= num_sms)
          ks = d > 0 ? static_cast<int>(std::ceil(est_p / std::max(est_d, 1.0))) : num_sms / pairs;
        static const int ks_env = getenv("SARATHI_PREFILL_KSPLIT") ? atoi(getenv("SARATHI_PREFILL_KSPLIT")) : 0;
        if (ks_env > 0) ks = ks_env;
        static const int ks_cap = getenv("SARATHI_PREFILL_KSPLIT_MAX") ? atoi(getenv("SARATHI_PREFILL_KSPLIT_MAX")) : 4;
        ks = std::min({ks, std::min(ks_cap, 8), first_tiles, std::max(1, num_sms / pairs)});
        if (static_cast<size_t>(pairs) * ks * 128 > pp_rows || pairs > pp_pairs) ks = 1;
        pa.ksplit = std::max(1, ks);
        pa.part_o = pp_o;
        pa.part_ml = pp_ml;
        pa.counters = pp_ctr;
      }
      if (xflags_try) {
        pa.done_flag = aflags + nkv_l;
        pa.done_cnt = acnt + nkv_l;
        pa.epoch = attn_epoch;
      }
      // with decodes in the batch, the chunk's attention overlaps the decode attention: by default
      // both run in the main stream as an "attention chain" (prefill, PDL-launched, waits for QKV
      // and then triggers the decode grid, whose CTAs wait for the prefill grid at their end), so
      // the prefill CTAs take their SMs first and no cross-stream fork / join is needed;
      // SARATHI_ATTN_CHAIN=0 puts the prefill on the high-priority side stream instead
      const bool side = d > 0 && !no_aux && !chain;
      cudaStream_t ps = side ? aux : stream;
      if (side) {
        SRET(check(cudaEventRecord(ev_fork, stream), "fork"));
        SRET(check(cudaStreamWaitEvent(aux, ev_fork, 0), "fork"));
      }
      ob = op_begin(ps);
      static const char* ptrace = getenv("SARATHI_PREFILL_TRACE");  // debug: stamps of one launch with p == N
      static bool ptraced = false;
      unsigned long long* trbuf = nullptr;
      if (ptrace && !ptraced && atoi(ptrace) == p && l == 1) {
        ptraced = true;
        cudaMalloc(&trbuf, 1024 * 8);
        cudaMemsetAsync(trbuf, 0, 1024 * 8, ps);
        pa.trace = trbuf;
        stamp_kernel<<<1, 1, 0, ps>>>(trbuf + 1000);
      }
      SRET(take_span(SARATHI_OP_PREFILL_ATTN, &pa.span_start, &pa.span_end));
      SRET(check(launch_prefill_attention(pa, &m_q, &kmap[l], &vmap[l], ps), "prefill attention"));
      if (trbuf) {
        unsigned long long hb[1024];
        cudaStreamSynchronize(ps);
        cudaMemcpy(hb, trbuf, sizeof(hb), cudaMemcpyDeviceToHost);
        const unsigned long long t0 = hb[254];
        for (int t = 0; t < 32 && hb[t * 8]; ++t) {
          fprintf(stderr, "prefill tile %2d:", t);
          for (int k = 0; k < 7; ++k) fprintf(stderr, " %8.3f", hb[t * 8 + k] ? (hb[t * 8 + k] - t0) * 1e-3 : -1.0);
          fprintf(stderr, "\n");
        }
        fprintf(stderr, "prefill last PV done %8.3f us\n", (hb[255] - t0) * 1e-3);
        unsigned long long s_min = ~0ull;
        for (int b = 0; b < 384 && hb[256 + 2 * b]; ++b) s_min = std::min(s_min, hb[256 + 2 * b]);
        fprintf(stderr, "prefill stream ready %8.3f us before the first CTA\n", (s_min - hb[1000]) * 1e-3);
        for (int b = 0; b < 384 && hb[256 + 2 * b]; ++b)
          fprintf(stderr, "prefill cta %3d: start %8.3f end %8.3f us\n", b, (hb[256 + 2 * b] - s_min) * 1e-3,
                  (hb[257 + 2 * b] - s_min) * 1e-3);
        cudaFree(trbuf);
      }
      op_end(SARATHI_OP_PREFILL_ATTN, ob, ps);
      ++launches;
      if (side) SRET(check(cudaEventRecord(ev_join, aux), "join"));
    }
    if (d > 0) {
      DecodeAttnArgs da;
      da.q = q;
      da.q_ld = q_dim_l;
      da.q_row0 = p;
      da.kcache = kpool[l];
      da.vcache = vpool[l];
      da.block_tables = d_dtab;
      da.ctx = d_ctx;
      da.max_blocks = max_blocks_per_req;
      da.d = d;
      da.n_q_local = nq_l;
      da.n_kv_local = nkv_l;
      da.head_dim = hd;
      da.block_size = block_size;
      da.scale = scale;
      int max_nblk = 0;
      for (int j = 0; j < d; ++j) max_nblk = std::max(max_nblk, (dec->positions[j] + 1 + block_size - 1) / block_size);
      // split the sequence (flash-decoding) by a small cost model in microseconds: whole waves of
      // 2-CTA-per-SM slots x (fixed per-CTA cost + blocks per split x per-block stream time), plus
      // the combine kernel when split.  13B TP1 (2560 CTAs) stays unsplit; a 70B TP-8 rank (26
      // requests x 1 KV head, 32 blocks) splits ~11 ways into one wave.
      const int base_ctas = d * nkv_l;
      const int slots = 2 * num_sms;
      int splits = 1;
      double best = 1e30;
      for (int sp = 1; sp <= max_nblk; ++sp) {
        const int bps = (max_nblk + sp - 1) / sp;
        const int n = (max_nblk + bps - 1) / bps;
        if (n != sp) continue;  // same partition as a smaller split count
        const long long ctas = static_cast<long long>(base_ctas) * n;
        const double waves = static_cast<double>((ctas + slots - 1) / slots);
        const double t = waves * (2.0 + 1.5 * bps) + (n > 1 ? 3.0 : 0.0);
        if (t < best - 1e-9) {
          best = t;
          splits = n;
        }
      }
      const size_t per_split = static_cast<size_t>(d) * nq_l * hd;
      splits = static_cast<int>(std::max<size_t>(1, std::min<size_t>(splits, part_cap / per_split)));
      da.blocks_per_split = (max_nblk + splits - 1) / splits;
      da.splits = (max_nblk + da.blocks_per_split - 1) / da.blocks_per_split;
      {
        const size_t blk = static_cast<size_t>(block_size) * hd * 2;  // K (or V) block bytes
        da.stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(4, (104 * 1024) / (2 * blk))));
        static const int st_env = getenv("SARATHI_DECODE_STAGES") ? atoi(getenv("SARATHI_DECODE_STAGES")) : 0;
        if (st_env >= 2) da.stages = st_env;  // experiment
      }
      static const int dec_dbg = getenv("SARATHI_DECODE_DBG") ? atoi(getenv("SARATHI_DECODE_DBG")) : 0;
      da.dbg = dec_dbg;
      static const int dec_nopdl = getenv("SARATHI_DECODE_NOPDL") ? atoi(getenv("SARATHI_DECODE_NOPDL")) : 0;
      da.no_pdl = (dec_nopdl == 1 && p > 0 && !no_aux) || dec_nopdl == 2;
      da.wait_at_end = chain;
      da.part_o = part_o;
      da.part_lse = part_lse;
      da.out = o;
      da.out_ld = q_dim_l;
      if (xflags_try && da.splits == 1) {
        da.head_flag = aflags;
        da.head_cnt = acnt;
        da.epoch = attn_epoch;
        xflags = true;
      }
      ob = op_begin();
      SRET(take_span(SARATHI_OP_DECODE_ATTN, &da.span_start, &da.span_end));
      SRET(check(launch_decode_attention(da, kmap[l], vmap[l], stream), "decode attention"));
      op_end(SARATHI_OP_DECODE_ATTN, ob);
      launches += da.splits > 1 ? 2 : 1;
      if (p > 0 && !no_aux && !chain) SRET(check(cudaStreamWaitEvent(stream, ev_join, 0), "join"));
    }
    if (use_chain) {
      ob = op_begin();
      SRET(run_chain(l, T, l + 1 < nl, d_pos, d_slot));
      op_end(SARATHI_OP_GEMM_CHAIN, ob);
      continue;
    }
    // O-projection (postproj) + residual / TP all-reduce
    EpiParams eo;
    if (world == 1) {
      eo.mode = EPI_ADD_F32;
      eo.out = h;
      eo.ldo = H;
    } else {
      eo.mode = EPI_STORE_BF16;
      eo.out = ar_target();
      eo.ldo = H;
    }
    if (xflags) {  // X = o: per KV head (G query heads x hd columns) + the chunk's rows
      eo.xflag = aflags;
      eo.xflag_cols = (nq_l / nkv_l) * hd;
      eo.xflag_n = nkv_l;
      eo.xflag2 = p > 0 ? aflags + nkv_l : nullptr;
      eo.xepoch = attn_epoch;
    }
    if (post_norm) set_pnorm(eo, w.g2);
    if (norm_flags) eo.done_ctr = gemm_done;
    ob = op_begin();
    SRET(gemm(w.m_o, H, q_dim_l, o, q_dim_l, T, eo, SARATHI_OP_GEMM_O));
    op_end(SARATHI_OP_GEMM_O, ob);
    if (world > 1) {
      ob = op_begin();
      SRET(allreduce());
      op_end(SARATHI_OP_ALLREDUCE, ob);
    }
    if (!norm_fused && !post_norm) {
    ob = op_begin();
    {
      unsigned long long *sp0, *sp1;
      SRET(take_span(SARATHI_OP_RMSNORM, &sp0, &sp1));
      NormFlags nf;
      if (norm_flags) flag_norm(nf);
      SRET(check(launch_rmsnorm(h, world > 1 ? pend : no_add, w.g2, a, nullptr, T, H, cfg.rms_eps, stream, sp0, sp1, nf),
                 "rmsnorm2"));
    }
    if (world > 1) SRET(ar_end());
    op_end(SARATHI_OP_RMSNORM, ob);
    ++launches;
    }
    // FFN
    EpiParams ef;
    if (norm_fused) set_norm(ef, w.g2);
    if (norm_flags) flag_x(ef);
    ef.mode = cfg.ffn_kind == SARATHI_FFN_SWIGLU ? EPI_SILU_MUL : EPI_GELU;
    ef.out = f;
    ef.ldo = h2_l;
    ob = op_begin();
    SRET(gemm(w.m_gu, gu_rows, H, a, H, T, ef, SARATHI_OP_GEMM_GATE_UP));
    op_end(SARATHI_OP_GEMM_GATE_UP, ob);
    EpiParams ed;
    if (world == 1) {
      ed.mode = EPI_ADD_F32;
      ed.out = h;
      ed.ldo = H;
    } else {
      ed.mode = EPI_STORE_BF16;
      ed.out = ar_target();
      ed.ldo = H;
    }
    normed_next = post_norm && l + 1 < nl;
    if (normed_next) set_pnorm(ed, layers[l + 1].g1);
    flag_next = norm_flags && l + 1 < nl;
    if (flag_next) ed.done_ctr = gemm_done;
    ob = op_begin();
    SRET(gemm(w.m_down, H, h2_l, f, h2_l, T, ed, SARATHI_OP_GEMM_DOWN));
    op_end(SARATHI_OP_GEMM_DOWN, ob);
    if (world > 1) {
      ob = op_begin();
      SRET(allreduce());
      op_end(SARATHI_OP_ALLREDUCE, ob);
      pending_ar = true;
    }
  }
  if (pending_ar && (dump_layers || !want_logits || all_rows)) {
    SRET(check(launch_residual_add(h, pend, T, H, stream), "residual add"));
    SRET(ar_end());
    ++launches;
    pending_ar = false;
  }
  SRET(dump_h(nl));
  if (want_logits) {
    ob = op_begin();
    // final norm on the R logit rows (adds the pending TP partial for exactly those rows)
    SRET(check(launch_rmsnorm(h, pending_ar ? pend : no_add, gf, af, d_rows, R, H, cfg.rms_eps, stream), "final norm"));
    if (pending_ar) SRET(ar_end());
    ++launches;
    const bool host_out = flags & SARATHI_LOGITS_HOST;
    float* target = host_out ? logits_dev : logits;
    EpiParams el;
    el.mode = EPI_STORE_F32;
    if (world == 1) {
      el.out = target;
      el.ldo = cfg.vocab;
      SRET(gemm(m_lm, vocab_l, H, af, H, R, el));
    } else {
      el.out = logits_local;
      el.ldo = vocab_l;
      SRET(gemm(m_lm, vocab_l, H, af, H, R, el));
      if (group) {
        SRET(local_allgather_f32(group, rank, logits_local, logits_gather, static_cast<size_t>(R) * vocab_l, stream));
      } else {
        ncclResult_t r = api->allGather(logits_local, logits_gather, static_cast<size_t>(R) * vocab_l, ncclFloat32,
                                        static_cast<ncclComm_t>(nccl), stream);
        if (r != ncclSuccess) return Status::err(SARATHI_ENCCL, "ncclAllGather failed");
      }
      SRET(check(launch_vocab_permute(logits_gather, target, world, R, vocab_l, cfg.vocab, stream), "permute"));
      ++launches;
    }
    op_end(SARATHI_OP_LM_HEAD, ob);
    if (host_out) {
      last_d2h = static_cast<int64_t>(R) * cfg.vocab * 4;
      SRET(check(cudaMemcpyAsync(logits, logits_dev, static_cast<size_t>(R) * cfg.vocab * 4, cudaMemcpyDeviceToHost, stream),
                 "D2H logits"));
      SRET(check(cudaStreamSynchronize(stream), "sync logits"));
    }
  }
  SRET(check(cudaGetLastError(), "launch"));
  // ---- state advance (a12) ----
  if (pre) cached[pre->req_id] += p;
  for (int j = 0; j < d; ++j) cached[dec->req_ids[j]] += 1;
  last_T = T;
  last_dumped = dump_layers;
  return Status::ok();
}

void Model::destroy() {
  if (stream) cudaStreamSynchronize(stream);
  if (nvls) nvls_teardown(*this);
  if (nccl) {
    NcclApi* api = nccl_api(nullptr);
    if (api) api->commDestroy(static_cast<ncclComm_t>(nccl));
    nccl = nullptr;
  }
  if (group) {
    local_group_leave(group, rank);
    group = nullptr;
  }
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
  ipc_opened.clear();
  for (void* p : allocations) cudaFree(p);
  allocations.clear();
  if (owns_stream && stream) cudaStreamDestroy(stream);
  owns_stream = false;
  if (aux) cudaStreamSynchronize(aux);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (aux) cudaStreamDestroy(aux);
  aux = nullptr;
  ev_fork = ev_join = nullptr;
  for (int i = 0; i < 2; ++i) {
    if (meta_host_buf[i]) cudaFreeHost(meta_host_buf[i]);
    if (meta_ev[i]) cudaEventDestroy(meta_ev[i]);
    meta_host_buf[i] = nullptr;
    meta_ev[i] = nullptr;
  }
}

}  // namespace sarathi

// Internal model state behind the sarathi_model handle.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sarathi.h"
#include "gemm.cuh"
#include "host_sched.hpp"
#include "kernels.cuh"

namespace sarathi {

struct Status {
  int code = SARATHI_OK;
  std::string msg;
  static Status ok() { return Status(); }
  static Status err(int c, std::string m) {
    Status s;
    s.code = c;
    s.msg = std::move(m);
    return s;
  }
};

// Local TP group (collective.cu): `world` handles on one device standing in for one process per GPU.
struct LocalGroup;
Status local_group_create(int world, int device, LocalGroup** out);
void local_group_destroy(LocalGroup* g);
Status local_group_join(LocalGroup* g, int rank, int world, int device);
void local_group_leave(LocalGroup* g, int rank);
// result = bf16(sum over ranks of partial) on every rank (ncclAllReduce semantics, out of place)
Status local_allreduce_bf16(LocalGroup* g, int rank, const __nv_bfloat16* partial, __nv_bfloat16* result, size_t count,
                            int num_sms, cudaStream_t st);
// dst[r * count ...] = rank r's src (ncclAllGather layout)
Status local_allgather_f32(LocalGroup* g, int rank, const float* src, float* dst, size_t count, cudaStream_t st);
// Fused all-reduce (NEXT-1) in a local group: register this rank's partial buffers / ready flags,
// read the peers' (valid once every rank has initialised), and order the streams around the
// consumer kernel (events + host barrier: the device-side flags are then always already set).
void local_group_register(LocalGroup* g, int rank, __nv_bfloat16* const arbuf[2], unsigned int* ready);
bool local_group_peers(LocalGroup* g, const __nv_bfloat16* peer_ar[2][8], unsigned int* peer_ready[8]);
Status local_fused_begin(LocalGroup* g, int rank, cudaStream_t st);
Status local_fused_end(LocalGroup* g, int rank, cudaStream_t st);
// Publish this rank's partial of all-reduce `epoch`: ready_r[rank] = epoch on every rank r
// (st.release.sys after a system fence; peer flags over NVLink / same device).
cudaError_t launch_signal_ready(unsigned int* const peer_ready[8], int rank, int world, unsigned int epoch,
                                cudaStream_t st);

struct LayerWeights {
  __nv_bfloat16* qkv = nullptr;   // [(nq_l + 2 nkv_l) hd][H]
  __nv_bfloat16* o = nullptr;     // [H][nq_l hd]
  __nv_bfloat16* gu = nullptr;    // [2 H2_l][H] gate/up interleaved in 16-row blocks (SwiGLU) | [H2_l][H] (GELU)
  __nv_bfloat16* down = nullptr;  // [H][H2_l]
  __nv_bfloat16* g1 = nullptr;    // [H]
  __nv_bfloat16* g2 = nullptr;    // [H]
  CUtensorMap m_qkv, m_o, m_gu, m_down;  // make_tmap_weight maps of the packed weights
};

struct Model {
  sarathi_model_config cfg{};
  int rank = 0, world = 1, device = 0;
  // pipeline parallelism (NEXT-4): this handle holds layers [l0, l0 + nl) of the L layers
  int pp_stage = 0, pp_stages = 1, l0 = 0, nl = 0;
  const float* pp_in = nullptr;  // stage > 0: the previous stage's residual stream [T][H] (device)
  cudaStream_t stream = nullptr;
  // side stream, used only with SARATHI_ATTN_CHAIN=0 (the default "attention chain" keeps both
  // attentions in the main stream): the chunked-prefill attention runs concurrently with the
  // decode attention of the same layer (fork after the QKV GEMM, join before the O GEMM)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int num_sms = 148;
  uint64_t seed = 0;
  // sharded sizes
  int nq_l = 0, nkv_l = 0, q_dim_l = 0, kv_dim_l = 0, qkv_rows = 0, h2_l = 0, gu_rows = 0, vocab_l = 0;
  // weights
  __nv_bfloat16* emb = nullptr;  // [V][H]
  __nv_bfloat16* gf = nullptr;   // [H]
  __nv_bfloat16* lm = nullptr;   // [vocab_l][H]
  CUtensorMap m_lm;
  CUtensorMap m_q;  // q buffer [Tmax][q_dim_l], box 128 x 64 (tcgen05 prefill attention)
  std::vector<LayerWeights> layers;
  std::vector<void*> allocations;
  float* rope_theta = nullptr;  // [hd/2][2] RoPE frequencies (fp64 -> fp32 hi + lo)
  // KV cache
  bool kv_ready = false;
  int64_t num_blocks = 0;
  int block_size = 0;
  int max_blocks_per_req = 0;
  std::vector<__nv_bfloat16*> kpool, vpool;
  std::vector<CUtensorMap> kmap, vmap;  // TMA maps of the pools (decode attention)
  BlockAllocator alloc;
  std::map<int64_t, int32_t> cached;
  // activations / workspaces (Tmax rows)
  int Tmax = 0;
  float* h = nullptr;
  __nv_bfloat16 *a = nullptr, *q = nullptr, *o = nullptr, *f = nullptr, *ar = nullptr, *af = nullptr;
  float* logits_dev = nullptr;     // [Tmax][V]   (host-output / TP staging)
  float* logits_local = nullptr;   // [Tmax][vocab_l]
  float* logits_gather = nullptr;  // [world][Tmax][vocab_l]
  float* gemm_ws = nullptr;
  size_t gemm_ws_floats = 0;
  int* gemm_counters = nullptr;
  float* part_o = nullptr;
  float* part_lse = nullptr;
  size_t part_cap = 0;  // floats in part_o
  // chunked-prefill key-split partials (PrefillAttnArgs::ksplit): O rows, (m, l), per-pair counters
  float* pp_o = nullptr;
  float* pp_ml = nullptr;
  int* pp_ctr = nullptr;
  size_t pp_rows = 0;  // 128-row x ksplit capacity of pp_o in rows of head_dim floats
  int pp_pairs = 0;    // counters
  int* meta_dev = nullptr;
  int* meta_host_buf[2] = {nullptr, nullptr};  // pinned, double-buffered
  cudaEvent_t meta_ev[2] = {nullptr, nullptr};
  int meta_flip = 0;
  size_t meta_ints = 0;
  float* dump = nullptr;     // [(L+1)][Tmax][H]
  int last_T = 0;
  bool last_dumped = false;
  std::vector<int32_t> last_slots;
  // caches
  std::map<std::tuple<int, int, int>, GemmPlan> plans;
  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> xmaps;
  // TP collectives: NCCL communicator (one process per GPU) or a local group (one device)
  void* nccl = nullptr;
  LocalGroup* group = nullptr;
  __nv_bfloat16* ar_red = nullptr;        // local group: all-reduce result buffer [Tmax][H]
  const __nv_bfloat16* ar_res = nullptr;  // buffer holding the latest all-reduce result (ar or ar_red)
  bool owns_stream = false;
  // fused TP all-reduce: the row-parallel GEMM writes its bf16 partial to
  // arbuf[epoch & 1] (peer-visible), signals the ranks' ready flags, and the consuming RMSNorm /
  // residual kernel sums every rank's partial over peer memory (one-shot all-reduce fused into
  // the consumer, no NCCL call).  Double buffering makes a separate "done reading" flag unneeded.
  bool tp_fused = false;
  __nv_bfloat16* arbuf[2] = {nullptr, nullptr};
  unsigned int* ready = nullptr;                 // [8] epochs published by each rank (this rank's copy)
  const __nv_bfloat16* peer_ar[2][8] = {};       // rank r's arbuf[b]
  unsigned int* peer_ready[8] = {};              // rank r's ready array
  bool peers_ok = false;
  unsigned int ar_epoch = 0;
  std::vector<void*> ipc_opened;                 // cudaIpcOpenMemHandle mappings (multi-process)
  // NVLS variant (nvls.cu, SARATHI_TP_NVLS=1): partials + flags in an NCCL symmetric window,
  // the consumer reads the rank sum through the window's multimem address
  bool tp_nvls = false;
  void* nvls = nullptr;                          // NvlsState
  const __nv_bfloat16* mm_ar[2] = {nullptr, nullptr};
  // layer chain (gemm_chain.cu, world == 1): O -> FFN1 -> FFN2 -> next layer's QKV in ONE launch,
  // tile-level flags instead of kernel boundaries, RMSNorm folded into finalisers + epilogue scales
  bool chain_on = false;
  __nv_bfloat16* a2 = nullptr;        // FFN1 input bf16(g2 * h), written by the O finalisers [Tmax][H]
  float* ss1 = nullptr;               // per-128-column sums of squares of h for the next QKV [H/128][Tmax]
  float* ss2 = nullptr;               // ... for FFN1
  unsigned* cflags = nullptr;         // O fin [nt_h] | FFN1 out [nt_gu] | FFN2 fin [nt_h] (epoch-valued)
  int* ccnt = nullptr;                // O fin [nt_h] | FFN2 fin [nt_h] | FFN1 arrive/written [2 nt_gu] | QKV [2 nt_qkv]
  int nt_qkv = 0;
  float* cscr = nullptr;              // split-tile scratch [Tmax][scr_ld] (zero between launches)
  int scr_ld = 0;
  int nt_h = 0, nt_gu = 0;            // 128-row tiles (rounded up to pair tiles)
  unsigned chain_epoch = 0;
  struct ChainPlanDev {
    ChainSchedule sch;
    int* dev = nullptr;  // segs | seg_off | need(O) | need(FFN2)
    ChainLaunch base;
    int need_o = 0, need_f2 = 0;  // offsets (ints) of the need arrays in dev
    int need_gu = 0, slab_gu = 0, need_qkv = 0, slab_qkv = 0;  // split whole-tile jobs
  };
  std::map<std::pair<int, int>, ChainPlanDev> chain_plans;  // (T, with next QKV)
  Status chain_plan(int T, bool with_qkv, const ChainPlanDev** out);
  Status run_chain(int l, int T, bool with_qkv, const int* d_pos, const int* d_slot);
  Status xmap(const void* X, int N, int K, int ldx, int box_rows, const CUtensorMap** out);
  // attention -> O projection handoff (EpiParams::xflag): per-KV-head completion flags of the decode
  // attention + the prefill attention's grid-completion flag, epoch-valued; counters zero between launches
  unsigned* aflags = nullptr;  // [n_kv_l] heads | [1] prefill done
  int* acnt = nullptr;         // [n_kv_l + 1]
  unsigned attn_epoch = 0;
  // fused RMSNorm prologue of the QKV / gate||up GEMMs (EpiParams::norm_*): grid-barrier counter
  // (monotonic) and the arrivals issued so far
  unsigned* norm_ctr = nullptr;
  unsigned norm_arrivals = 0;
  // flag-chained RMSNorm (SARATHI_NORM_FLAGS): residual-add GEMM CTAs -> gemm_done, rmsnorm CTAs ->
  // norm_done (monotonic; targets = all arrivals so far)
  unsigned* gemm_done = nullptr;
  unsigned gemm_done_arrivals = 0;
  unsigned* norm_done = nullptr;
  unsigned norm_done_arrivals = 0;
  int64_t launches = 0;
  // I/O accounting and per-op timers
  int64_t last_h2d = 0, last_d2h = 0;
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending_ops;
  double op_ms[SARATHI_NUM_OPS] = {0};
  int64_t op_count[SARATHI_NUM_OPS] = {0};
  // in-kernel device spans of profiled GEMM launches (first CTA start -> last CTA end, globaltimer)
  static constexpr int kSpanCap = 4096;
  unsigned long long* span_buf = nullptr;  // [kSpanCap] starts (atomicMin) | [kSpanCap] ends (atomicMax)
  std::vector<int> span_ops;
  double op_kms[SARATHI_NUM_OPS] = {0};
  int64_t op_kcount[SARATHI_NUM_OPS] = {0};
  cudaEvent_t op_begin(cudaStream_t s = nullptr);
  void op_end(int op, cudaEvent_t b, cudaStream_t s = nullptr);
  Status collect_op_times();

  // host_tensors: NULL (generate from seed) or the logical weights, see sarathi_init_model
  Status init(const sarathi_model_config& c, const sarathi_dist& d, uint64_t seed, const void* const* host_tensors);
  Status alloc_kv(int64_t num_blocks, int32_t block_size);
  Status ipc_exchange();
  Status run(const sarathi_prefill_chunk* pre, const sarathi_decode_set* dec, float* logits, int32_t flags);
  void destroy();

  // helpers
  Status gemm(const CUtensorMap& mw, int M, int K, const void* X, int ldx, int N, const EpiParams& ep, int op = -1);
  // profiling: a (start, end) device-span slot for one launch of op (null pointers when off / full)
  Status take_span(int op, unsigned long long** start, unsigned long long** end);
  Status check(cudaError_t e, const char* what);
  template <typename T>
  Status dalloc(T** p, size_t count);
  Status dalloc_padded(__nv_bfloat16** p, int rows, int cols);  // tile-major GEMM weight, rows -> x128
};

int nccl_unique_id(void* out128, std::string* err);
Status nvls_setup(Model& m);
void nvls_teardown(Model& m);

}  // namespace sarathi

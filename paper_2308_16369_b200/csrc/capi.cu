// extern "C" boundary (include/sarathi.h): argument checks, status codes, thread-local errors.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/sarathi.h"
#include "model.hpp"

struct sarathi_model {
  sarathi::Model m;
};
struct sarathi_sched {
  sarathi::Scheduler* s = nullptr;
  sarathi::PlanOut last;
};

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int from(const sarathi::Status& s) {
  if (s.code != SARATHI_OK) g_err = s.msg;
  return s.code;
}
}  // namespace

extern "C" {

const char* sarathi_last_error(void) { return g_err.c_str(); }

int sarathi_nccl_unique_id(void* out128) {
  if (!out128) return fail(SARATHI_EINVAL, "nccl_unique_id: NULL");
  std::string err;
  const int r = sarathi::nccl_unique_id(out128, &err);
  if (r != SARATHI_OK) return fail(r, err);
  return SARATHI_OK;
}

int sarathi_local_group_create(int32_t world, int32_t device, sarathi_local_group** out) {
  if (!out) return fail(SARATHI_EINVAL, "local_group_create: NULL");
  sarathi::LocalGroup* g = nullptr;
  const sarathi::Status s = sarathi::local_group_create(world, device, &g);
  if (s.code != SARATHI_OK) return from(s);
  *out = reinterpret_cast<sarathi_local_group*>(g);
  return SARATHI_OK;
}

void sarathi_local_group_destroy(sarathi_local_group* g) {
  sarathi::local_group_destroy(reinterpret_cast<sarathi::LocalGroup*>(g));
}

int sarathi_init_model(const sarathi_model_config* cfg, const sarathi_dist* dist, uint64_t weight_seed,
                       const void* const* host_tensors, sarathi_model** out) {
  if (!cfg || !dist || !out) return fail(SARATHI_EINVAL, "init_model: NULL argument");
  auto* h = new (std::nothrow) sarathi_model();
  if (!h) return fail(SARATHI_EINVAL, "init_model: out of host memory");
  const sarathi::Status s = h->m.init(*cfg, *dist, weight_seed, host_tensors);
  if (s.code != SARATHI_OK) {
    h->m.destroy();
    delete h;
    return from(s);
  }
  *out = h;
  return SARATHI_OK;
}

void sarathi_destroy(sarathi_model* m) {
  if (!m) return;
  m->m.destroy();
  delete m;
}

int sarathi_alloc_kv(sarathi_model* m, int64_t num_blocks, int32_t block_size) {
  if (!m) return fail(SARATHI_EINVAL, "alloc_kv: NULL model");
  return from(m->m.alloc_kv(num_blocks, block_size));
}

int sarathi_kv_bytes_per_token(const sarathi_model* m, int64_t* out) {
  if (!m || !out) return fail(SARATHI_EINVAL, "kv_bytes_per_token: NULL");
  *out = 2ll * m->m.nl * m->m.nkv_l * m->m.cfg.head_dim * 2;  // this handle's layers
  return SARATHI_OK;
}

int sarathi_max_batch(const sarathi_model* m, int32_t tokens_per_request, int64_t reserve_bytes, int32_t* B_out) {
  if (!m || !B_out || tokens_per_request < 1) return fail(SARATHI_EINVAL, "max_batch: bad argument");
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return fail(SARATHI_ECUDA, "cudaMemGetInfo failed");
  const double num = static_cast<double>(fr) - static_cast<double>(reserve_bytes);
  const double mkv = 2.0 * m->m.nl * m->m.nkv_l * m->m.cfg.head_dim * 2;
  *B_out = num <= 0 ? 0 : static_cast<int32_t>(num / (tokens_per_request * mkv));
  return SARATHI_OK;
}

int sarathi_request_alloc(sarathi_model* m, int64_t req_id, int32_t max_tokens) {
  if (!m) return fail(SARATHI_EINVAL, "request_alloc: NULL model");
  auto& M = m->m;
  if (!M.kv_ready) return fail(SARATHI_ESTATE, "request_alloc: alloc_kv not called");
  if (max_tokens < 1 || max_tokens > M.cfg.max_seq_len) return fail(SARATHI_EINVAL, "request_alloc: max_tokens out of range");
  if (M.alloc.has(req_id)) return fail(SARATHI_EINVAL, "request_alloc: id already allocated");
  if (!M.alloc.alloc(req_id, max_tokens)) return fail(SARATHI_ENOKV, "request_alloc: not enough free KV blocks");
  M.cached[req_id] = 0;
  return SARATHI_OK;
}

int sarathi_request_free(sarathi_model* m, int64_t req_id) {
  if (!m) return fail(SARATHI_EINVAL, "request_free: NULL model");
  if (!m->m.alloc.has(req_id)) return fail(SARATHI_EUNKNOWN_REQ, "request_free: unknown request");
  m->m.alloc.free(req_id);
  m->m.cached.erase(req_id);
  return SARATHI_OK;
}

int sarathi_request_cached_len(const sarathi_model* m, int64_t req_id, int32_t* len_out) {
  if (!m || !len_out) return fail(SARATHI_EINVAL, "request_cached_len: NULL");
  auto it = m->m.cached.find(req_id);
  if (it == m->m.cached.end()) return fail(SARATHI_EUNKNOWN_REQ, "request_cached_len: unknown request");
  *len_out = it->second;
  return SARATHI_OK;
}

int sarathi_request_truncate(sarathi_model* m, int64_t req_id, int32_t new_len) {
  if (!m) return fail(SARATHI_EINVAL, "request_truncate: NULL model");
  auto it = m->m.cached.find(req_id);
  if (it == m->m.cached.end()) return fail(SARATHI_EUNKNOWN_REQ, "request_truncate: unknown request");
  if (new_len < 0 || new_len > it->second) return fail(SARATHI_EINVAL, "request_truncate: new_len > cached length");
  it->second = new_len;
  return SARATHI_OK;
}

int sarathi_stage_input(sarathi_model* m, const float* h_dev) {
  if (!m || !h_dev) return fail(SARATHI_EINVAL, "stage_input: NULL");
  if (m->m.pp_stage == 0) return fail(SARATHI_EINVAL, "stage_input: the first pipeline stage embeds its tokens");
  m->m.pp_in = h_dev;
  return SARATHI_OK;
}

int sarathi_stage_output(const sarathi_model* m, const float** h_dev, int32_t* T_out) {
  if (!m || !h_dev || !T_out) return fail(SARATHI_EINVAL, "stage_output: NULL");
  *h_dev = m->m.h;
  *T_out = m->m.last_T;
  return SARATHI_OK;
}

int sarathi_last_io_bytes(const sarathi_model* m, int64_t* h2d, int64_t* d2h) {
  if (!m || !h2d || !d2h) return fail(SARATHI_EINVAL, "last_io_bytes: NULL");
  *h2d = m->m.last_h2d;
  *d2h = m->m.last_d2h;
  return SARATHI_OK;
}

int sarathi_set_profiling(sarathi_model* m, int32_t enable) {
  if (!m) return fail(SARATHI_EINVAL, "set_profiling: NULL");
  m->m.profiling = enable != 0;
  return SARATHI_OK;
}

int sarathi_op_times(sarathi_model* m, double* ms_out, int64_t* counts_out, int32_t n, int32_t reset) {
  if (!m || !ms_out || !counts_out || n < SARATHI_NUM_OPS) return fail(SARATHI_EINVAL, "op_times: bad argument");
  const sarathi::Status s = m->m.collect_op_times();
  if (s.code != SARATHI_OK) return from(s);
  for (int i = 0; i < SARATHI_NUM_OPS; ++i) {
    ms_out[i] = m->m.op_ms[i];
    counts_out[i] = m->m.op_count[i];
    if (reset) {
      m->m.op_ms[i] = 0;
      m->m.op_count[i] = 0;
    }
  }
  return SARATHI_OK;
}

int sarathi_op_kernel_times(sarathi_model* m, double* ms_out, int64_t* counts_out, int32_t n, int32_t reset) {
  if (!m || !ms_out || !counts_out || n < SARATHI_NUM_OPS) return fail(SARATHI_EINVAL, "op_kernel_times: bad argument");
  const sarathi::Status s = m->m.collect_op_times();
  if (s.code != SARATHI_OK) return from(s);
  for (int i = 0; i < SARATHI_NUM_OPS; ++i) {
    ms_out[i] = m->m.op_kms[i];
    counts_out[i] = m->m.op_kcount[i];
    if (reset) {
      m->m.op_kms[i] = 0;
      m->m.op_kcount[i] = 0;
    }
  }
  return SARATHI_OK;
}

int sarathi_run_hybrid_batch(sarathi_model* m, const sarathi_prefill_chunk* prefill, const sarathi_decode_set* decodes,
                             float* logits, int32_t flags) {
  if (!m) return fail(SARATHI_EINVAL, "run_hybrid_batch: NULL model");
  return from(m->m.run(prefill, decodes, logits, flags));
}

int sarathi_debug_slot_mapping(const sarathi_model* m, int32_t* out, int32_t cap, int32_t* T_out) {
  if (!m || !T_out) return fail(SARATHI_EINVAL, "debug_slot_mapping: NULL");
  const auto& s = m->m.last_slots;
  *T_out = static_cast<int32_t>(s.size());
  if (out) {
    if (cap < static_cast<int32_t>(s.size())) return fail(SARATHI_EINVAL, "debug_slot_mapping: cap too small");
    std::memcpy(out, s.data(), s.size() * sizeof(int32_t));
  }
  return SARATHI_OK;
}

int sarathi_debug_block_table(const sarathi_model* m, int64_t req_id, int32_t* out, int32_t cap, int32_t* n_out) {
  if (!m || !n_out) return fail(SARATHI_EINVAL, "debug_block_table: NULL");
  if (!m->m.alloc.has(req_id)) return fail(SARATHI_EUNKNOWN_REQ, "debug_block_table: unknown request");
  const auto& t = m->m.alloc.table(req_id);
  *n_out = static_cast<int32_t>(t.size());
  if (out) {
    if (cap < static_cast<int32_t>(t.size())) return fail(SARATHI_EINVAL, "debug_block_table: cap too small");
    std::memcpy(out, t.data(), t.size() * sizeof(int32_t));
  }
  return SARATHI_OK;
}

int sarathi_debug_hidden(const sarathi_model* m, int32_t layer, float* host_out) {
  if (!m || !host_out) return fail(SARATHI_EINVAL, "debug_hidden: NULL");
  const auto& M = m->m;
  if (!M.last_dumped || !M.dump) return fail(SARATHI_ESTATE, "debug_hidden: last batch not run with DUMP_LAYERS");
  if (layer < -1 || layer >= M.nl) return fail(SARATHI_EINVAL, "debug_hidden: layer out of range (this stage's layers)");
  cudaStreamSynchronize(M.stream);
  const size_t n = static_cast<size_t>(M.last_T) * M.cfg.hidden;
  if (cudaMemcpy(host_out, M.dump + static_cast<size_t>(layer + 1) * M.Tmax * M.cfg.hidden, n * 4,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(SARATHI_ECUDA, "debug_hidden: copy failed");
  return SARATHI_OK;
}

int sarathi_debug_kv(const sarathi_model* m, int32_t layer, int64_t req_id, int32_t pos0, int32_t n, uint16_t* host_k,
                     uint16_t* host_v) {
  if (!m || !host_k || !host_v) return fail(SARATHI_EINVAL, "debug_kv: NULL");
  const auto& M = m->m;
  if (!M.kv_ready || layer < 0 || layer >= M.nl) return fail(SARATHI_EINVAL, "debug_kv: bad layer/state");
  if (!M.alloc.has(req_id)) return fail(SARATHI_EUNKNOWN_REQ, "debug_kv: unknown request");
  if (pos0 < 0 || n < 0 || pos0 + n > M.alloc.reserved(req_id)) return fail(SARATHI_EINVAL, "debug_kv: range");
  cudaStreamSynchronize(M.stream);
  const int hd = M.cfg.head_dim, bs = M.block_size;
  // copy whole [n_kv_local][bs][hd] blocks, then gather the requested positions on the host
  const size_t blk_elems = static_cast<size_t>(M.nkv_l) * bs * hd;
  std::vector<uint16_t> kb(blk_elems), vb(blk_elems);
  const auto& table = M.alloc.table(req_id);
  int cur_blk = -1;
  for (int i = 0; i < n; ++i) {
    const int pos = pos0 + i;
    const int bi = pos / bs;
    if (bi != cur_blk) {
      const size_t off = static_cast<size_t>(table[bi]) * blk_elems;
      if (cudaMemcpy(kb.data(), M.kpool[layer] + off, blk_elems * 2, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(vb.data(), M.vpool[layer] + off, blk_elems * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(SARATHI_ECUDA, "debug_kv: copy failed");
      cur_blk = bi;
    }
    for (int hh = 0; hh < M.nkv_l; ++hh) {
      const size_t src = (static_cast<size_t>(hh) * bs + pos % bs) * hd;
      const size_t dst = (static_cast<size_t>(i) * M.nkv_l + hh) * hd;
      std::memcpy(host_k + dst, kb.data() + src, hd * 2);
      std::memcpy(host_v + dst, vb.data() + src, hd * 2);
    }
  }
  return SARATHI_OK;
}

int sarathi_debug_weight(const sarathi_model* m, int32_t layer, int32_t tensor, int64_t offset, int64_t count,
                         uint16_t* host_out) {
  if (!m || !host_out || offset < 0 || count < 0) return fail(SARATHI_EINVAL, "debug_weight: bad argument");
  const auto& M = m->m;
  const __nv_bfloat16* src = nullptr;
  int rows = 0, cols = 0;
  bool packed = true;  // GEMM weights live in the tile-major layout; report the logical [rows][cols] view
  const int H = M.cfg.hidden;
  if (tensor < 16) {
    if (layer < 0 || layer >= M.nl) return fail(SARATHI_EINVAL, "debug_weight: layer (this stage's layers)");
    const auto& w = M.layers[layer];
    switch (tensor) {
      case 0: src = w.qkv; rows = M.qkv_rows; cols = H; break;
      case 1: src = w.o; rows = H; cols = M.q_dim_l; break;
      case 2: src = w.gu; rows = M.gu_rows; cols = H; break;
      case 3: src = w.down; rows = H; cols = M.h2_l; break;
      case 4: src = w.g1; rows = 1; cols = H; packed = false; break;
      case 5: src = w.g2; rows = 1; cols = H; packed = false; break;
      default: return fail(SARATHI_EINVAL, "debug_weight: tensor");
    }
  } else {
    switch (tensor) {
      case 16: src = M.emb; rows = M.cfg.vocab; cols = H; packed = false; break;
      case 17: src = M.gf; rows = 1; cols = H; packed = false; break;
      case 18: src = M.lm; rows = M.vocab_l; cols = H; break;
      default: return fail(SARATHI_EINVAL, "debug_weight: tensor");
    }
  }
  const size_t total = static_cast<size_t>(rows) * cols;
  if (!src) return fail(SARATHI_EINVAL, "debug_weight: tensor not held by this pipeline stage");
  if (static_cast<size_t>(offset + count) > total) return fail(SARATHI_EINVAL, "debug_weight: range");
  cudaStreamSynchronize(M.stream);
  if (!packed) {
    if (cudaMemcpy(host_out, src + offset, count * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(SARATHI_ECUDA, "debug_weight: copy failed");
    return SARATHI_OK;
  }
  const size_t padded = static_cast<size_t>((rows + 127) / 128) * 128 * cols;
  std::vector<uint16_t> buf(padded);
  if (cudaMemcpy(buf.data(), src, padded * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(SARATHI_ECUDA, "debug_weight: copy failed");
  for (int64_t i = 0; i < count; ++i) {
    const int64_t li = offset + i;
    host_out[i] = buf[sarathi::packed_weight_index(static_cast<int>(li / cols), static_cast<int>(li % cols), cols)];
  }
  return SARATHI_OK;
}

int sarathi_launch_count(const sarathi_model* m, int64_t* out) {
  if (!m || !out) return fail(SARATHI_EINVAL, "launch_count: NULL");
  *out = m->m.launches;
  return SARATHI_OK;
}

int sarathi_shard_map(const sarathi_model_config* cfg, int32_t rank, int32_t world, int32_t layer, int32_t tensor,
                      int32_t* tau, float* scale, int64_t* base, int32_t cap, int32_t* rows, int32_t* cols) {
  if (!cfg || !rows || !cols || world < 1 || rank < 0 || rank >= world)
    return fail(SARATHI_EINVAL, "shard_map: bad argument");
  std::vector<int> t;
  std::vector<float> sc;
  std::vector<long long> b;
  sarathi::ShardDims d;
  if (!sarathi::shard_map(cfg->n_layers, cfg->hidden, cfg->n_heads, cfg->n_kv_heads, cfg->head_dim, cfg->ffn_hidden,
                          cfg->vocab, cfg->ffn_kind, rank, world, layer, tensor, &t, &sc, &b, &d))
    return fail(SARATHI_EINVAL, "shard_map: bad tensor id");
  *rows = d.rows;
  *cols = d.cols;
  if (tau || scale || base) {
    if (cap < d.rows) return fail(SARATHI_EINVAL, "shard_map: cap too small");
    for (int r = 0; r < d.rows; ++r) {
      if (tau) tau[r] = t[r];
      if (scale) scale[r] = sc[r];
      if (base) base[r] = b[r];
    }
  }
  return SARATHI_OK;
}

// ---- scheduler ----
int sarathi_sched_create(int32_t B, int32_t C, int32_t policy, int32_t tile_adjust, int64_t num_blocks,
                         int32_t block_size, sarathi_sched** out) {
  if (!out || B < 1 || C < 1 || policy < 0 || policy > 2 || num_blocks < 0 || block_size < 1)
    return fail(SARATHI_EINVAL, "sched_create: bad argument");
  if (tile_adjust < 0 || tile_adjust > 2) return fail(SARATHI_EINVAL, "sched_create: tile_adjust must be 0, 1 or 2");
  if (tile_adjust == 1 && C <= B - 1) return fail(SARATHI_EINVAL, "sched_create: tile-adjusted chunk C-(B-1) must be >= 1");
  auto* s = new (std::nothrow) sarathi_sched();
  if (!s) return fail(SARATHI_EINVAL, "sched_create: out of memory");
  s->s = new sarathi::Scheduler(B, C, policy, tile_adjust, num_blocks, block_size);
  *out = s;
  return SARATHI_OK;
}

void sarathi_sched_destroy(sarathi_sched* s) {
  if (!s) return;
  delete s->s;
  delete s;
}

int sarathi_sched_submit(sarathi_sched* s, int64_t req_id, int32_t P, int32_t D, int32_t arrival_iter) {
  if (!s) return fail(SARATHI_EINVAL, "sched_submit: NULL");
  std::string err;
  const int rc = s->s->submit(req_id, P, D, arrival_iter, &err);
  if (rc != SARATHI_OK) return fail(rc, err);
  return SARATHI_OK;
}

int sarathi_sched_next(sarathi_sched* s, sarathi_plan* plan, int64_t* dec_req, int32_t* dec_pos, int64_t* admitted,
                       int32_t cap) {
  if (!s || !plan) return fail(SARATHI_EINVAL, "sched_next: NULL");
  // admitted and decodes are each at most B: check before next() mutates the scheduler
  if (cap < s->s->B()) return fail(SARATHI_EINVAL, "sched_next: cap must be >= B");
  sarathi::PlanOut p;
  const bool have = s->s->next(&p);
  plan->iteration = p.iteration;
  plan->prefill_req = p.prefill_req;
  plan->prefill_start = p.prefill_start;
  plan->prefill_len = p.prefill_len;
  plan->n_decodes = static_cast<int32_t>(p.decodes.size());
  plan->n_admitted = static_cast<int32_t>(p.admitted.size());
  for (size_t i = 0; i < p.decodes.size(); ++i) {
    if (dec_req) dec_req[i] = p.decodes[i].first;
    if (dec_pos) dec_pos[i] = p.decodes[i].second;
  }
  for (size_t i = 0; i < p.admitted.size(); ++i)
    if (admitted) admitted[i] = p.admitted[i];
  return have ? 1 : 0;
}

int sarathi_sched_complete(sarathi_sched* s, int64_t* finished, int32_t cap, int32_t* n_finished) {
  if (!s || !n_finished) return fail(SARATHI_EINVAL, "sched_complete: NULL");
  // at most B requests run, so at most B finish: check before complete() mutates the scheduler
  if (finished && cap < s->s->B()) return fail(SARATHI_EINVAL, "sched_complete: cap must be >= B");
  const auto fin = s->s->complete();
  *n_finished = static_cast<int32_t>(fin.size());
  for (size_t i = 0; i < fin.size(); ++i)
    if (finished) finished[i] = fin[i];
  return SARATHI_OK;
}

int sarathi_sched_idle_step(sarathi_sched* s) {
  if (!s) return fail(SARATHI_EINVAL, "sched_idle_step: NULL");
  s->s->idle_step();
  return SARATHI_OK;
}

int sarathi_sched_done(const sarathi_sched* s, int32_t* done) {
  if (!s || !done) return fail(SARATHI_EINVAL, "sched_done: NULL");
  *done = s->s->done() ? 1 : 0;
  return SARATHI_OK;
}

int sarathi_sched_block_table(const sarathi_sched* s, int64_t req_id, int32_t* out, int32_t cap, int32_t* n_out) {
  if (!s || !n_out) return fail(SARATHI_EINVAL, "sched_block_table: NULL");
  const auto& a = s->s->allocator();
  if (!a.has(req_id)) return fail(SARATHI_EUNKNOWN_REQ, "sched_block_table: unknown request");
  const auto& t = a.table(req_id);
  *n_out = static_cast<int32_t>(t.size());
  if (out) {
    if (cap < static_cast<int32_t>(t.size())) return fail(SARATHI_EINVAL, "sched_block_table: cap");
    std::memcpy(out, t.data(), t.size() * sizeof(int32_t));
  }
  return SARATHI_OK;
}

int sarathi_token_capacity(int32_t T, int32_t* capacity, int32_t* n_tiles, int32_t* n_mma) {
  if (T < 1 || !capacity) return fail(SARATHI_EINVAL, "token_capacity: bad argument");
  const sarathi::TokenTiling t = sarathi::gemm_token_tiling(T);
  *capacity = t.capacity();
  if (n_tiles) *n_tiles = t.n_tiles;
  if (n_mma) *n_mma = t.n_mma;
  return SARATHI_OK;
}

int sarathi_chunk_advice(int32_t C, int32_t d, int32_t remaining, int32_t* p_out) {
  if (C < 1 || d < 0 || remaining < 1 || !p_out) return fail(SARATHI_EINVAL, "chunk_advice: bad argument");
  *p_out = sarathi::b200_chunk(C, d, remaining);
  return SARATHI_OK;
}

int sarathi_chain_schedule(int32_t njobs, const int32_t* pm_tiles, const int32_t* KB, const int32_t* split,
                           const int32_t* dep_shift, const double* e_done, int32_t pairs, double e_add, double e_fin,
                           int32_t* seg_off, int32_t* segs, int32_t cap, int32_t* n_segs, double* makespan) {
  if (njobs < 1 || njobs > 8 || !pm_tiles || !KB || !split || !dep_shift || !e_done || pairs < 1 || !seg_off || !segs ||
      !n_segs || cap < 0)
    return fail(SARATHI_EINVAL, "chain_schedule: bad argument");
  std::vector<sarathi::ChainJobShape> jobs(njobs);
  for (int j = 0; j < njobs; ++j) {
    if (pm_tiles[j] < 1 || KB[j] < 1) return fail(SARATHI_EINVAL, "chain_schedule: empty job");
    jobs[j] = {pm_tiles[j], KB[j], split[j] != 0, dep_shift[j], e_done[j]};
  }
  const sarathi::ChainSchedule sc = sarathi::schedule_chain(jobs, pairs, e_add, e_fin);
  const int n = static_cast<int>(sc.segs.size() / 4);
  if (n > cap) return fail(SARATHI_EINVAL, "chain_schedule: cap too small");
  std::copy(sc.seg_off.begin(), sc.seg_off.end(), seg_off);
  std::copy(sc.segs.begin(), sc.segs.end(), segs);
  *n_segs = n;
  if (makespan) *makespan = sc.makespan;
  return SARATHI_OK;
}

// ---- kernel-level ops ----
int sarathi_op_gemm(const void* W, const void* X, void* out, int32_t M, int32_t N, int32_t K, int32_t mode,
                    int32_t force_splits, void* stream) {
  using namespace sarathi;
  const bool prepacked = (mode & SARATHI_GEMM_W_PACKED) != 0;
  mode &= ~SARATHI_GEMM_W_PACKED;
  if (!W || !X || !out || M < 8 || M % 8 || N < 1 || K < 64 || K % 64 || mode < 0 || mode > 4)
    return fail(SARATHI_EINVAL, "op_gemm: bad argument (M % 8 == 0, K % 64 == 0, mode 0..4)");
  if (mode == EPI_SILU_MUL && M % 128) return fail(SARATHI_EINVAL, "op_gemm: SiLU mode needs M % 128 == 0");
  static float* ws = nullptr;
  static int* ctr = nullptr;
  static size_t ws_floats = static_cast<size_t>(64) << 20;  // lower half slot partials, upper half red.add
  if (!ws) {
    if (cudaMalloc(&ws, ws_floats * 4) != cudaSuccess || cudaMalloc(&ctr, (1 << 16) * 4) != cudaSuccess ||
        cudaMemset(ctr, 0, (1 << 16) * 4) != cudaSuccess ||
        cudaMemset(ws + ws_floats / 2, 0, ws_floats / 2 * 4) != cudaSuccess)
      return fail(SARATHI_ECUDA, "op_gemm: workspace allocation failed");
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemmPlan pl = plan_gemm(M, N, K, sms, ws_floats, force_splits, mode == EPI_ADD_F32);
  if (const char* st_env = getenv("SARATHI_GEMM_STAGES")) {  // timing experiments: fewer ring stages
    const int want = atoi(st_env);
    if (want >= 2 && want < pl.stages) {
      pl.smem -= static_cast<size_t>(pl.stages - want) * (16384 + static_cast<size_t>(pl.bn / 2) * 128);
      pl.stages = want;
    }
  }
  // pack W into the library's tile-major layout (the layout init_model generates weights in)
  static __nv_bfloat16* wp = nullptr;
  static size_t wp_elems = 0;
  const size_t need = static_cast<size_t>((M + 127) / 128) * 128 * K;
  if (need > wp_elems) {
    if (wp) cudaFree(wp);
    wp = nullptr;
    if (cudaMalloc(&wp, need * 2) != cudaSuccess) return fail(SARATHI_ECUDA, "op_gemm: pack buffer allocation failed");
    wp_elems = need;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!prepacked && (cudaMemsetAsync(wp, 0, need * 2, st) != cudaSuccess ||
                     launch_pack_weight(static_cast<const __nv_bfloat16*>(W), wp, M, K, st) != cudaSuccess))
    return fail(SARATHI_ECUDA, "op_gemm: weight packing failed");
  CUtensorMap mw, mx, mx2;
  if (!make_tmap_weight(&mw, prepacked ? W : wp, M, K) || !make_tmap_bf16(&mx, X, N, K, K, pl.box_rows) ||
      !make_tmap_bf16(&mx2, X, N, K, K, pl.box_rows2))
    return fail(SARATHI_ECUDA, "op_gemm: tensor map encode failed");
  EpiParams ep;
  ep.mode = mode;
  ep.out = out;
  ep.ldo = mode == EPI_SILU_MUL ? M / 2 : M;
  ep.ws = ws;
  ep.ws_red = ws + ws_floats / 2;
  ep.counters = ctr;
  if (const char* d = getenv("SARATHI_GEMM_DBG")) ep.dbg = atoi(d);
  static unsigned long long* trace = nullptr;
  const bool tracing = getenv("SARATHI_GEMM_TRACE") != nullptr;
  if (tracing) {
    if (!trace) cudaMalloc(&trace, 4096 * 8);
    cudaMemsetAsync(trace, 0, 4096 * 8, st);
    ep.trace = trace;
  }
  const cudaError_t e = launch_gemm(mw, mx, mx2, pl, ep, st);
  if (tracing) {
    cudaStreamSynchronize(st);
    dump_gemm_trace(trace, pl);
  }
  if (e != cudaSuccess) return fail(SARATHI_ECUDA, std::string("op_gemm: ") + cudaGetErrorString(e));
  return SARATHI_OK;
}

int sarathi_op_pack_weight(const void* W, void* out, int32_t rows, int32_t cols, void* stream) {
  if (!W || !out || rows < 1 || cols < 64 || cols % 64) return fail(SARATHI_EINVAL, "op_pack_weight: bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t n = static_cast<size_t>((rows + 127) / 128) * 128 * cols;
  if (cudaMemsetAsync(out, 0, n * 2, st) != cudaSuccess ||
      sarathi::launch_pack_weight(static_cast<const __nv_bfloat16*>(W), static_cast<__nv_bfloat16*>(out), rows, cols,
                                  st) != cudaSuccess)
    return fail(SARATHI_ECUDA, "op_pack_weight: launch failed");
  return SARATHI_OK;
}

int sarathi_op_rmsnorm(const float* h, const void* g, void* out, int32_t R, int32_t H, float eps, void* stream) {
  if (!h || !g || !out || R < 0 || H < 4 || H % 4) return fail(SARATHI_EINVAL, "op_rmsnorm: bad argument");
  const cudaError_t e = sarathi::launch_rmsnorm(const_cast<float*>(h), nullptr, static_cast<const __nv_bfloat16*>(g),
                                                static_cast<__nv_bfloat16*>(out), nullptr, R, H, eps,
                                                static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SARATHI_ECUDA, std::string("op_rmsnorm: ") + cudaGetErrorString(e));
  return SARATHI_OK;
}

}  // extern "C"

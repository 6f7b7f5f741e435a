// Host-side KV block allocator and scheduler (see host_sched.hpp).
#include "host_sched.hpp"

#include <algorithm>
#include <cmath>

#include "../../include/sarathi.h"

namespace sarathi {

TokenTiling gemm_token_tiling(int T) {
  TokenTiling t;
  T = std::max(T, 1);
  t.n_tiles = (T + 511) / 512;
  const int per = (T + t.n_tiles - 1) / t.n_tiles;
  if (per <= 256) {
    t.n_mma = 1;
    t.bn = std::max(16, (per + 15) / 16 * 16);
  } else {
    t.n_mma = 2;
    t.bn = (per + 31) / 32 * 32;
  }
  return t;
}

int b200_chunk(int C, int d, int remaining) {
  const int T = C + d;
  int p = gemm_token_tiling(T).capacity() - d;
  for (int b : {256, 512})
    if (T > b && T - b <= C / 8 && b - d >= 1) {
      p = b - d;
      break;
    }
  return std::max(1, std::min(p, remaining));
}

BlockAllocator::BlockAllocator(int64_t num_blocks, int32_t block_size)
    : num_blocks_(num_blocks), block_size_(block_size) {
  for (int64_t b = 0; b < num_blocks; ++b) free_.insert(static_cast<int32_t>(b));
}

bool BlockAllocator::alloc(int64_t req, int64_t max_tokens) {
  const int64_t n = blocks_for(max_tokens);
  if (n > static_cast<int64_t>(free_.size())) return false;
  std::vector<int32_t> t;
  t.reserve(n);
  auto it = free_.begin();
  for (int64_t i = 0; i < n; ++i) t.push_back(*it++);  // lowest ids first (std::set is ordered)
  free_.erase(free_.begin(), it);
  tables_[req] = std::move(t);
  reserved_[req] = max_tokens;
  return true;
}

void BlockAllocator::free(int64_t req) {
  auto it = tables_.find(req);
  if (it == tables_.end()) return;
  for (int32_t b : it->second) free_.insert(b);
  tables_.erase(it);
  reserved_.erase(req);
}

Scheduler::Scheduler(int32_t B, int32_t C, int32_t policy, int32_t tile_adjust, int64_t num_blocks, int32_t block_size)
    : B_(B), C_(C), policy_(policy), tile_adjust_(tile_adjust), alloc_(num_blocks, block_size) {}

int Scheduler::submit(int64_t req, int32_t P, int32_t D, int32_t arrival, std::string* err) {
  if (reqs_.count(req) || P < 1 || D < 0) {
    if (err) *err = "sched_submit: duplicate id or bad P/D";
    return SARATHI_EINVAL;
  }
  if (alloc_.blocks_for(static_cast<int64_t>(P) + D) > alloc_.num_blocks()) {
    if (err) *err = "sched_submit: the P+D KV reservation exceeds the whole block pool (never admissible)";
    return SARATHI_ENOKV;
  }
  Req r;
  r.id = req;
  r.P = P;
  r.D = D;
  r.arrival = arrival;
  reqs_.emplace(req, r);
  return SARATHI_OK;
}

std::vector<Scheduler::Req*> Scheduler::running() {
  std::vector<Req*> v;
  for (auto& kv : reqs_)
    if (kv.second.admitted && !kv.second.finished) v.push_back(&kv.second);
  std::sort(v.begin(), v.end(), [](const Req* a, const Req* b) { return a->admit_seq < b->admit_seq; });
  return v;
}

bool Scheduler::done() const {
  for (const auto& kv : reqs_)
    if (!kv.second.finished) return false;
  return true;
}

bool Scheduler::next(PlanOut* out) {
  PlanOut plan;
  plan.iteration = iteration_;
  // admission: FCFS by (arrival, id), strict (stop at the first that does not fit)
  std::vector<Req*> run = running();
  if (!(policy_ == REQUEST_LEVEL && !run.empty())) {
    std::vector<Req*> pend;
    for (auto& kv : reqs_)
      if (!kv.second.admitted && kv.second.arrival <= iteration_) pend.push_back(&kv.second);
    std::sort(pend.begin(), pend.end(), [](const Req* a, const Req* b) {
      return a->arrival != b->arrival ? a->arrival < b->arrival : a->id < b->id;
    });
    int32_t nrun = static_cast<int32_t>(run.size());
    for (Req* r : pend) {
      if (nrun >= B_ || !alloc_.can_alloc(static_cast<int64_t>(r->P) + r->D)) break;
      alloc_.alloc(r->id, static_cast<int64_t>(r->P) + r->D);
      r->admitted = true;
      r->admit_seq = admit_counter_++;
      plan.admitted.push_back(r->id);
      ++nrun;
    }
    run = running();
  }
  Req* cand = nullptr;
  for (Req* r : run)
    if (r->prefill_done < r->P) {
      cand = r;
      break;
    }
  std::vector<Req*> dec;
  for (Req* r : run)
    if (r->prefill_done == r->P && r->decode_done < r->D) dec.push_back(r);
  const size_t cap = static_cast<size_t>(cand ? B_ - 1 : B_);
  if (cand) {
    const int32_t remaining = cand->P - cand->prefill_done;
    int32_t len;
    if (policy_ == ORCA_BEST || policy_ == REQUEST_LEVEL)
      len = remaining;
    else if (tile_adjust_ == 2)  // decodes riding in THIS batch
      len = b200_chunk(C_, static_cast<int>(std::min(dec.size(), cap)), remaining);
    else
      len = std::min(tile_adjust_ == 1 ? C_ - (B_ - 1) : C_, remaining);
    plan.prefill_req = cand->id;
    plan.prefill_start = cand->prefill_done;
    plan.prefill_len = len;
    if (policy_ == REQUEST_LEVEL) dec.clear();
  }
  for (size_t i = 0; i < dec.size() && i < cap; ++i)
    plan.decodes.emplace_back(dec[i]->id, dec[i]->P + dec[i]->decode_done);
  if (!cand && plan.decodes.empty()) {
    // admissions (if any) stay; nothing to run
    *out = plan;
    have_plan_ = false;
    return false;
  }
  last_ = plan;
  have_plan_ = true;
  *out = plan;
  return true;
}

std::vector<int64_t> Scheduler::complete() {
  std::vector<int64_t> fin;
  if (!have_plan_) return fin;
  if (last_.prefill_req >= 0) {
    Req& r = reqs_.at(last_.prefill_req);
    r.prefill_done += last_.prefill_len;
    if (r.prefill_done == r.P && r.D == 0) fin.push_back(r.id);
  }
  for (const auto& d : last_.decodes) {
    Req& r = reqs_.at(d.first);
    r.decode_done += 1;
    if (r.decode_done == r.D) fin.push_back(r.id);
  }
  for (int64_t id : fin) {
    reqs_.at(id).finished = true;
    alloc_.free(id);
  }
  have_plan_ = false;
  ++iteration_;
  return fin;
}

namespace {
constexpr int kWQ = 0, kWK = 1, kWV = 2, kWO = 3, kWG = 4, kWU = 5, kWD = 6;
constexpr int kEmbTau = 1 << 20, kWlmTau = (1 << 20) + 2;
float weight_scale(double sigma) { return static_cast<float>(std::sqrt(3.0) * sigma / 16777216.0); }
}  // namespace

bool shard_map(int n_layers, int hidden, int n_heads, int n_kv_heads, int head_dim, int ffn_hidden, int vocab,
               int ffn_kind, int rank, int world, int layer, int tensor, std::vector<int>* tau,
               std::vector<float>* scale, std::vector<long long>* base, ShardDims* dims) {
  const int H = hidden, hd = head_dim;
  const int q_dim_l = n_heads / world * hd, kv_dim_l = n_kv_heads / world * hd;
  const int h2_l = ffn_hidden / world, vocab_l = vocab / world;
  const double s_in = 1.0 / std::sqrt(static_cast<double>(H));
  const double depth = 1.0 / std::sqrt(2.0 * n_layers);
  const double s_o = depth / std::sqrt(static_cast<double>(n_heads) * hd);
  const double s_d = depth / std::sqrt(static_cast<double>(ffn_hidden));
  int rows = 0, cols = 0;
  switch (tensor) {
    case 0: rows = q_dim_l + 2 * kv_dim_l; cols = H; break;
    case 1: rows = H; cols = q_dim_l; break;
    case 2: rows = ffn_kind == 0 ? 2 * h2_l : h2_l; cols = H; break;
    case 3: rows = H; cols = h2_l; break;
    case 16: rows = vocab; cols = H; break;
    case 18: rows = vocab_l; cols = H; break;
    default: return false;
  }
  tau->assign(rows, 0);
  scale->assign(rows, 0.f);
  base->assign(rows, 0);
  for (int r = 0; r < rows; ++r) {
    int kind = 0;
    long long b = 0;
    double sig = s_in;
    switch (tensor) {
      case 0: {  // [q_r ; k_r ; v_r]: the rank's heads of the logical Wq, Wk, Wv
        // inside each head, packed row 32j + l (l < 16) is dim 16j + l and row 32j + 16 + l is its
        // rotate-half partner hd/2 + 16j + l (gemm.cu: RoPE is a warp-local shuffle)
        int rr = r;
        if (r < q_dim_l) {
          kind = kWQ;
        } else if (r < q_dim_l + kv_dim_l) {
          kind = kWK;
          rr = r - q_dim_l;
        } else {
          kind = kWV;
          rr = r - q_dim_l - kv_dim_l;
        }
        const int head = rr / hd, pr = rr % hd, slab = pr / 32, l = pr % 32;
        const int d = (l < 16 ? 0 : hd / 2) + 16 * slab + (l % 16);
        const long long lrow = static_cast<long long>(rank) * (kind == kWQ ? q_dim_l : kv_dim_l) + head * hd + d;
        b = lrow * H;
        break;
      }
      case 1:  // row-parallel: columns rank*q_dim_l .. of the logical [H][n_heads*hd]
        kind = kWO;
        sig = s_o;
        b = static_cast<long long>(r) * n_heads * hd + static_cast<long long>(rank) * q_dim_l;
        break;
      case 2: {  // gate||up interleaved in 16-row blocks (SwiGLU) or W1 (GELU)
        long long fl = r;
        kind = kWG;
        if (ffn_kind == 0) {
          const int blk = r / 32, w2 = r % 32;
          kind = w2 < 16 ? kWG : kWU;
          fl = static_cast<long long>(blk) * 16 + (w2 % 16);
        }
        b = (static_cast<long long>(rank) * h2_l + fl) * H;
        break;
      }
      case 3:  // row-parallel down
        kind = kWD;
        sig = s_d;
        b = static_cast<long long>(r) * ffn_hidden + static_cast<long long>(rank) * h2_l;
        break;
      case 16:
        (*tau)[r] = kEmbTau;
        (*scale)[r] = weight_scale(1.0);
        (*base)[r] = static_cast<long long>(r) * H;
        continue;
      case 18:
        (*tau)[r] = kWlmTau;
        (*scale)[r] = weight_scale(s_in);
        (*base)[r] = (static_cast<long long>(rank) * vocab_l + r) * H;
        continue;
    }
    (*tau)[r] = 16 * layer + kind;
    (*scale)[r] = weight_scale(sig);
    (*base)[r] = b;
  }
  dims->rows = rows;
  dims->cols = cols;
  return true;
}

}  // namespace sarathi

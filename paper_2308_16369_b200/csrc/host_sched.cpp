// Host-side KV block allocator and scheduler (see host_sched.hpp).
#include "host_sched.hpp"

#include <algorithm>

namespace sarathi {

BlockAllocator::BlockAllocator(int64_t num_blocks, int32_t block_size)
    : num_blocks_(num_blocks), block_size_(block_size) {
  for (int64_t b = 0; b < num_blocks; ++b) free_.insert(static_cast<int32_t>(b));
}

bool BlockAllocator::alloc(int64_t req, int32_t max_tokens) {
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

Scheduler::Scheduler(int32_t B, int32_t C, int32_t policy, bool tile_adjust, int64_t num_blocks, int32_t block_size)
    : B_(B), C_(C), policy_(policy), tile_adjust_(tile_adjust), alloc_(num_blocks, block_size) {}

bool Scheduler::submit(int64_t req, int32_t P, int32_t D, int32_t arrival, std::string* err) {
  if (reqs_.count(req) || P < 1 || D < 0) {
    if (err) *err = "sched_submit: duplicate id or bad P/D";
    return false;
  }
  Req r;
  r.id = req;
  r.P = P;
  r.D = D;
  r.arrival = arrival;
  reqs_.emplace(req, r);
  return true;
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
      alloc_.alloc(r->id, r->P + r->D);
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
  if (cand) {
    int32_t c_eff;
    if (policy_ == ORCA_BEST || policy_ == REQUEST_LEVEL)
      c_eff = cand->P;
    else
      c_eff = tile_adjust_ ? C_ - (B_ - 1) : C_;
    plan.prefill_req = cand->id;
    plan.prefill_start = cand->prefill_done;
    plan.prefill_len = std::min(c_eff, cand->P - cand->prefill_done);
    if (policy_ == REQUEST_LEVEL) dec.clear();
  }
  const size_t cap = static_cast<size_t>(cand ? B_ - 1 : B_);
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

}  // namespace sarathi

// Host-side KV block allocator and scheduler (see host_sched.hpp).
#include "host_sched.hpp"

#include <algorithm>
#include <array>
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
  for (int b : {512})  // (the T = 256 step, one -> two UMMAs per k-step, is gone since the k-block issue fix)
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


ChainSchedule schedule_chain(const std::vector<ChainJobShape>& jobs, int P, double e_add, double e_fin, int min_seg,
                             bool split_whole) {
  ChainSchedule out;
  P = std::max(1, P);
  std::vector<double> f(P, 0.0);  // time each pair's MMA pipe becomes free
  std::vector<double> g(P, 0.0);  // time each pair's epilogue warps become free
  std::vector<std::vector<std::array<int, 4>>> per(P);
  std::vector<double> prev_ready;  // previous job: time each 128-row tile is published
  out.need.resize(jobs.size());
  using Assign = std::vector<std::array<int, 4>>;  // (pair, tile, k0, k1) in execution order per pair
  for (size_t j = 0; j < jobs.size(); ++j) {
    const ChainJobShape& J = jobs[j];
    const int KB = J.KB, PT = J.pm_tiles;
    std::vector<double> dep(KB, 0.0);
    if (J.dep_shift >= 0 && j > 0)
      for (int kb = 0; kb < KB; ++kb) {
        const size_t q = static_cast<size_t>(kb >> J.dep_shift);
        dep[kb] = q < prev_ready.size() ? prev_ready[q] : 0.0;
      }
    // a segment's mainloop: one unit per k-block, each k-block no earlier than its input
    auto run = [&](double t, int kb0, int kb1) {
      for (int kb = kb0; kb < kb1; ++kb) t = std::max(t, dep[kb]) + 1.0;
      return t;
    };
    // simulate an assignment on top of the current pair timelines: returns the time the job's last
    // tile is published; a tile with several contributors (split) is published after the last
    // contributor's epilogue (split residual job: + e_fin; split whole-tile job: + e_done)
    struct Sim {
      std::vector<double> f, g, ready;
      double end = 0.0;
    };
    auto simulate = [&](const Assign& as) {
      Sim r{f, g, std::vector<double>(2 * static_cast<size_t>(PT), 0.0)};
      std::vector<int> cnt(PT, 0);
      for (const auto& x : as) ++cnt[x[1]];
      std::vector<double> tile_end(PT, 0.0);
      for (const auto& x : as) {
        const double t = run(r.f[x[0]], x[2], x[3]);
        r.f[x[0]] = t;
        const bool whole = cnt[x[1]] == 1 && !J.split;
        const double e = std::max(t, r.g[x[0]]) + (whole ? J.e_done : e_add);
        r.g[x[0]] = e;
        tile_end[x[1]] = std::max(tile_end[x[1]], e);
      }
      for (int pt = 0; pt < PT; ++pt) {
        const double extra = J.split ? e_fin : (cnt[pt] > 1 ? J.e_done : 0.0);
        r.ready[2 * pt] = r.ready[2 * pt + 1] = tile_end[pt] + extra;
        r.end = std::max(r.end, r.ready[2 * pt]);
      }
      return r;
    };
    // water-filling of tiles [t0, PT) of the k-range [bk0, bk1): contiguous tile-major unit ranges
    // over the pairs' effective free times max(free, ready) so that every pair ends together
    auto waterfill = [&](const std::vector<double>& free_t, double bready, int t0, int bk0, int bk1) {
      const int len = bk1 - bk0;
      const long long U = static_cast<long long>(PT - t0) * len;
      Assign as;
      if (U <= 0) return as;
      std::vector<double> eff(P);
      for (int c = 0; c < P; ++c) eff[c] = std::max(free_t[c], bready);
      std::vector<int> order(P);
      for (int c = 0; c < P; ++c) order[c] = c;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return eff[x] < eff[y]; });
      int m = P;
      double T_end = 0.0;
      for (; m >= 1; --m) {
        double S = 0.0;
        for (int i = 0; i < m; ++i) S += eff[order[i]];
        T_end = (static_cast<double>(U) + S) / m;
        if (m == 1 || T_end >= eff[order[m - 1]]) break;
      }
      std::vector<long long> budget(m, 0);
      double cum = 0.0;
      long long given = 0;
      for (int i = 0; i < m; ++i) {
        cum += T_end - eff[order[i]];
        const long long upto = (i == m - 1) ? U : std::min<long long>(U, std::llround(cum));
        budget[i] = std::max<long long>(0, upto - given);
        given += budget[i];
      }
      // too-short ranges cost a whole epilogue: fold into a neighbour (and at most ~16 contributors
      // per tile and band)
      const long long shortest = std::max<long long>(min_seg, (len + 15) / 16);
      for (int i = 0; i < m; ++i)
        if (budget[i] > 0 && budget[i] < shortest) {
          int k = i + 1;
          if (k >= m)
            for (k = i - 1; k > 0 && budget[k] == 0; --k) {
            }
          if (k >= 0 && k != i) {
            budget[k] += budget[i];
            budget[i] = 0;
          }
        }
      int rpt = t0, rk = bk0;
      for (int i = 0; i < m; ++i) {
        long long n = budget[i];
        while (n > 0 && rpt < PT) {
          const int take = static_cast<int>(std::min<long long>(n, bk1 - rk));
          as.push_back({order[i], rpt, rk, rk + take});
          n -= take;
          rk += take;
          if (rk == bk1) {
            ++rpt;
            rk = bk0;
          }
        }
      }
      return as;
    };
    // tile-aligned split of tiles [t0, PT): each tile's k-range in n equal parts, LPT over the pairs
    auto aligned = [&](const std::vector<double>& free_t, double bready, int t0, int bk0, int bk1, int n) {
      const int len = bk1 - bk0;
      std::vector<std::array<int, 3>> parts;
      for (int pt = t0; pt < PT; ++pt)
        for (int q = 0; q < n; ++q)
          parts.push_back({pt, bk0 + static_cast<int>(static_cast<long long>(len) * q / n),
                           bk0 + static_cast<int>(static_cast<long long>(len) * (q + 1) / n)});
      std::stable_sort(parts.begin(), parts.end(),
                       [](const std::array<int, 3>& x, const std::array<int, 3>& y) { return x[2] - x[1] > y[2] - y[1]; });
      Assign as;
      std::vector<double> load(P);
      for (int c = 0; c < P; ++c) load[c] = std::max(free_t[c], bready);
      for (const auto& pr : parts) {
        int c = 0;
        for (int k = 1; k < P; ++k)
          if (load[k] < load[c]) c = k;
        as.push_back({c, pr[0], pr[1], pr[2]});
        load[c] += pr[2] - pr[1];
      }
      return as;
    };
    Assign best;
    Sim best_sim;
    bool have = false;
    auto consider = [&](const Assign& as) {
      Sim r = simulate(as);
      if (!have || r.end < best_sim.end - 1e-9) {
        best = as;
        best_sim = r;
        have = true;
      }
    };
    if (!J.split) {
      // whole tiles only; or `w` whole waves then the remaining tiles split (stream-K remainder);
      // or every tile split
      double dready = 0.0;
      for (int kb = 0; kb < KB; ++kb) dready = std::max(dready, dep[kb]);
      for (int w = PT / P; split_whole && w >= 0; --w) {
        Assign as;
        std::vector<double> ft(f);
        const int nwhole = (w == PT / P && PT % P == 0) ? PT : w * P;
        for (int pt = 0; pt < nwhole; ++pt) {  // whole tiles, LPT by free time
          const int c = static_cast<int>(std::min_element(ft.begin(), ft.end()) - ft.begin());
          as.push_back({c, pt, 0, KB});
          ft[c] = run(ft[c], 0, KB);
        }
        if (nwhole < PT) {
          Assign rest = waterfill(ft, dready, nwhole, 0, KB);
          as.insert(as.end(), rest.begin(), rest.end());
          for (int n = 1; n <= std::max(1, P / std::max(1, PT - nwhole)); ++n) {
            Assign al(as.begin(), as.begin() + nwhole);
            Assign r2 = aligned(ft, dready, nwhole, 0, KB, n);
            al.insert(al.end(), r2.begin(), r2.end());
            consider(al);
          }
        }
        consider(as);
      }
      {  // all whole tiles, LPT
        Assign as;
        std::vector<double> ft(f);
        for (int pt = 0; pt < PT; ++pt) {
          const int c = static_cast<int>(std::min_element(ft.begin(), ft.end()) - ft.begin());
          as.push_back({c, pt, 0, KB});
          ft[c] = run(ft[c], 0, KB);
        }
        consider(as);
      }
    } else {
      // residual job: per band (contiguous k-ranges whose inputs are published within `tol`),
      // in readiness order, the better of water-filling and tile-aligned splits
      const double tol = 4.0;
      std::vector<std::pair<int, int>> bands;
      for (int k0 = 0, kb = 1; kb <= KB; ++kb)
        if (kb == KB || std::fabs(dep[kb] - dep[k0]) > tol) {
          // a band of fewer than 8 k-blocks would only produce short segments: merge it
          if (!bands.empty() && (kb - k0 < 8 || bands.back().second - bands.back().first < 8))
            bands.back().second = kb;
          else
            bands.push_back({k0, kb});
          k0 = kb;
        }
      std::stable_sort(bands.begin(), bands.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
        return dep[x.first] < dep[y.first];
      });
      Assign all;
      std::vector<double> ft(f);
      for (const auto& band : bands) {
        double bready = 0.0;
        for (int kb = band.first; kb < band.second; ++kb) bready = std::max(bready, dep[kb]);
        Assign bb;
        double bend = 1e300;
        std::vector<Assign> cands;
        cands.push_back(waterfill(ft, bready, 0, band.first, band.second));
        for (int n = 1; n <= std::max(1, P / PT) && n <= band.second - band.first; ++n)
          cands.push_back(aligned(ft, bready, 0, band.first, band.second, n));
        for (const auto& c : cands) {
          Assign trial(all);
          trial.insert(trial.end(), c.begin(), c.end());
          const Sim r = simulate(trial);
          if (r.end < bend - 1e-9) {
            bend = r.end;
            bb = c;
          }
        }
        all.insert(all.end(), bb.begin(), bb.end());
        for (const auto& x : bb) ft[x[0]] = run(ft[x[0]], x[2], x[3]);
      }
      consider(all);
    }
    // commit: per-pair segments (a pair's consecutive ranges of one tile merge), contributor counts
    out.need[j].assign(PT, 0);
    for (const auto& x : best) {
      auto& v = per[x[0]];
      if (!v.empty() && v.back()[0] == static_cast<int>(j) && v.back()[1] == x[1] && v.back()[3] == x[2]) {
        v.back()[3] = x[3];
      } else {
        v.push_back({static_cast<int>(j), x[1], x[2], x[3]});
        ++out.need[j][x[1]];
      }
    }
    f = best_sim.f;
    g = best_sim.g;
    out.job_end.push_back(best_sim.end);
    prev_ready = best_sim.ready;
  }
  out.seg_off.assign(P + 1, 0);
  for (int c = 0; c < P; ++c) {
    out.seg_off[c + 1] = out.seg_off[c] + static_cast<int>(per[c].size());
    for (const auto& s : per[c]) out.segs.insert(out.segs.end(), s.begin(), s.end());
  }
  out.makespan = out.job_end.empty() ? 0.0 : out.job_end.back();
  for (double x : f) out.makespan = std::max(out.makespan, x);
  return out;
}

}  // namespace sarathi

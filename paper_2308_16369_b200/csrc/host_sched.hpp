// Host-side KV block allocator and decode-maximal batching scheduler (pure C++, no CUDA).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace sarathi {

// Token tiling of the swap-AB tcgen05 GEMM (gemm.cu plan_gemm uses exactly this): a batch of T
// tokens is cut into n_tiles = ceil(T / 512) token tiles of per = ceil(T / n_tiles) tokens; a tile
// of per <= 256 tokens is ONE UMMA per k-step of N = 16 * ceil(per / 16) (TMEM double-buffered),
// a wider one TWO UMMAs of N = bn / 2 with bn = 32 * ceil(per / 32).  capacity = bn * n_tiles is
// the number of token columns the GEMM computes anyway (the padding is free).
struct TokenTiling {
  int n_tiles = 1, bn = 16, n_mma = 1;
  int capacity() const { return bn * n_tiles; }
};
TokenTiling gemm_token_tiling(int T);

// B200 analogue of the paper's tile-quantization chunk rule (§4.4: the chunk is
// trimmed to C - (B-1) so chunk + decodes fills 256 tokens exactly, because crossing a 128-token
// tile boundary costs a whole extra tile).  Here the token quantum is the UMMA N granularity (16/32)
// and the cost step is at T = 512 (a second token tile re-streams the weights); the step at T = 256
// (one -> two UMMAs per k-step) disappeared with the one-asm k-block issue (reading O-23,
// profiles/r02_chunk_sweep_13b_s3.txt).  Given the configured chunk C, the batch's decode count d and
// the request's remaining prompt tokens:
//   * T = C + d just past the step b = 512 (T - b <= C / 8): trim, p = b - d;
//   * otherwise fill the padded tile: p = capacity(C + d) - d (>= C; those columns are computed anyway);
//   p = min(p, remaining), at least 1.
int b200_chunk(int C, int d, int remaining);

// Paged KV block allocator: a request reserves ceil(max_tokens / bs) blocks up front (the paper
// pre-allocates KV per maximum sequence length, §4.5), lowest-free-block-first
// (reading O-17) so the tables are deterministic and identical on every TP rank.
class BlockAllocator {
 public:
  BlockAllocator() = default;
  BlockAllocator(int64_t num_blocks, int32_t block_size);
  int64_t num_blocks() const { return num_blocks_; }
  int32_t block_size() const { return block_size_; }
  int64_t blocks_for(int64_t max_tokens) const { return (max_tokens + block_size_ - 1) / block_size_; }
  bool can_alloc(int64_t max_tokens) const { return blocks_for(max_tokens) <= static_cast<int64_t>(free_.size()); }
  bool has(int64_t req) const { return tables_.count(req) != 0; }
  // returns false if it does not fit
  bool alloc(int64_t req, int64_t max_tokens);
  void free(int64_t req);
  const std::vector<int32_t>& table(int64_t req) const { return tables_.at(req); }
  int64_t reserved(int64_t req) const { return reserved_.at(req); }
  int64_t free_blocks() const { return static_cast<int64_t>(free_.size()); }
  // slot = table[pos / bs] * bs + pos % bs
  int64_t slot(int64_t req, int32_t pos) const {
    const auto& t = tables_.at(req);
    return static_cast<int64_t>(t[pos / block_size_]) * block_size_ + pos % block_size_;
  }

 private:
  int64_t num_blocks_ = 0;
  int32_t block_size_ = 1;
  std::set<int32_t> free_;
  std::map<int64_t, std::vector<int32_t>> tables_;
  std::map<int64_t, int64_t> reserved_;
};

struct PlanOut {
  int32_t iteration = 0;
  int64_t prefill_req = -1;
  int32_t prefill_start = 0, prefill_len = 0;
  std::vector<std::pair<int64_t, int32_t>> decodes;  // (req, position)
  std::vector<int64_t> admitted;
};

// Decode-maximal batching (§4.3) with the paper's comparison policies
// (request-level baseline P:L26, Orca best case P:L104).  Mirrors the policy statement in
// include/sarathi.h; the Python twin in oracle/sched.py is an independent implementation.
class Scheduler {
 public:
  enum Policy { SARATHI = 0, ORCA_BEST = 1, REQUEST_LEVEL = 2 };
  // tile_adjust: 0 literal chunk C; 1 the paper's C - (B-1); 2 b200_chunk(C, d, remaining)
  Scheduler(int32_t B, int32_t C, int32_t policy, int32_t tile_adjust, int64_t num_blocks, int32_t block_size);
  // SARATHI_OK, SARATHI_EINVAL (duplicate id / P < 1 / D < 0) or SARATHI_ENOKV (the P+D
  // reservation needs more blocks than the whole pool: it could never be admitted and, with strict
  // FCFS, would block every later request forever)
  int submit(int64_t req, int32_t P, int32_t D, int32_t arrival, std::string* err);
  int32_t B() const { return B_; }
  // true if a plan was formed
  bool next(PlanOut* out);
  std::vector<int64_t> complete();
  void idle_step() { ++iteration_; }
  bool done() const;
  const BlockAllocator& allocator() const { return alloc_; }

 private:
  struct Req {
    int64_t id;
    int32_t P, D, arrival;
    int32_t prefill_done = 0, decode_done = 0;
    bool admitted = false, finished = false;
    int64_t admit_seq = -1;
  };
  std::vector<Req*> running();
  int32_t B_, C_, policy_;
  int32_t tile_adjust_;
  BlockAllocator alloc_;
  std::map<int64_t, Req> reqs_;
  int32_t iteration_ = 0;
  int64_t admit_counter_ = 0;
  bool have_plan_ = false;
  PlanOut last_;
};

// Megatron tensor-parallel shard of one packed weight (§2.3): for every row r of the
// rank-local packed tensor, the generator tensor id tau[r], fp32 scale[r] and the flat index base[r]
// of element (r, 0) in the LOGICAL tensor (element (r, c) is base[r] + c).  tensor: 0 qkv
// (column-parallel [q_r; k_r; v_r]), 1 o (row-parallel), 2 gate||up (column-parallel, 16-row
// interleave) / W1, 3 down (row-parallel), 16 embedding (replicated), 18 LM head (vocab-parallel).
// Host-only; returns false on a bad tensor id.
struct ShardDims {
  int rows = 0, cols = 0;
};
bool shard_map(int n_layers, int hidden, int n_heads, int n_kv_heads, int head_dim, int ffn_hidden, int vocab,
               int ffn_kind, int rank, int world, int layer, int tensor, std::vector<int>* tau,
               std::vector<float>* scale, std::vector<long long>* base, ShardDims* dims);

// ---------------------------------------------------------------------------
// Layer-chain schedule (gemm_chain.cu).  A chain is a sequence of GEMM jobs of one hybrid batch
// executed by ONE persistent launch of CTA pairs, job j+1 consuming job j's output tile by tile
// (dependency flags instead of kernel boundaries): O-proj -> FFN1 -> FFN2 -> next layer's QKV.
// Work is cut into segments (job, 256-row pair tile, k-block range); a whole-tile job (an epilogue
// that needs the full K sum: SiLU / GELU / RoPE) gets whole tiles, a split job (residual add,
// red.add into h) any k-range.  The schedule is a list schedule over a per-pair timeline in
// k-block units: whole tiles go to the earliest-free pair, a split job's units are ordered by the
// readiness of the k-blocks they consume (bands), then tile-major, and handed out as contiguous
// ranges so every pair ends at the same predicted time (water-filling over the pairs' free times).
struct ChainJobShape {
  int pm_tiles = 0;   // 256-row pair tiles
  int KB = 0;         // k-blocks of 64
  bool split = false; // residual-add job (any k-range per segment)
  int dep_shift = -1; // X k-block kb needs the previous job's 128-row tile kb >> dep_shift (-1: none)
  double e_done = 0;  // epilogue latency until the output tile is published (k-block units)
};
struct ChainSchedule {
  std::vector<int> seg_off;             // [pairs + 1] segment range of every pair
  std::vector<int> segs;                // 4 ints per segment: job, pair tile, kb0, kb1
  std::vector<std::vector<int>> need;   // per job, per pair tile: number of segments (split jobs)
  std::vector<double> job_end;          // predicted time the last tile of each job is published
  double makespan = 0;                  // predicted (k-block units)
};
// e_add: red.add epilogue of a split segment; e_fin: finalisation of a split tile after its last
// contributor (k-block units).  min_seg: split ranges shorter than this merge into a neighbour.
// split_whole: whole-tile jobs may also be split (contributors reduce through scratch slabs; the
// last one finishes the tile).  Measured slower than whole tiles on every shape tried (DESIGN.md
// §6: the last contributor's scratch reads are L2 round trips on the critical path), so opt-in.
ChainSchedule schedule_chain(const std::vector<ChainJobShape>& jobs, int pairs, double e_add, double e_fin,
                             int min_seg = 4, bool split_whole = true);

}  // namespace sarathi

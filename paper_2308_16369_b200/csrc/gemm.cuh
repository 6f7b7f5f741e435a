// Host-visible declarations of the tcgen05 GEMM (see gemm.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sarathi {

enum EpiMode : int {
  EPI_STORE_BF16 = 0,  // out[t, m] = bf16(acc)
  EPI_STORE_F32 = 1,   // out[t, m] = acc (fp32)
  EPI_ADD_F32 = 2,     // out[t, m] += acc (fp32 residual stream, fused residual add)
  EPI_SILU_MUL = 3,    // gate/up interleaved in 16-row blocks: out[t, f] = bf16(silu(g) * u)
  EPI_GELU = 4,        // out[t, m] = bf16(gelu_tanh(acc))
  EPI_QKV_ROPE = 5,    // RoPE(q,k) at pos[t]; q -> out; k,v -> paged KV cache at slot[t]
};

struct EpiParams {
  int mode = EPI_STORE_BF16;
  void* out = nullptr;
  long long ldo = 0;  // row stride of `out` in elements
  // EPI_QKV_ROPE
  const int* pos = nullptr;
  const int* slot = nullptr;
  const float* rope_theta = nullptr;  // [head_dim/2][2]: theta_i = base^(-2i/hd) as fp32 hi, lo
  void* kcache = nullptr;  // bf16 [num_blocks][n_kv_local][block_size][head_dim]
  void* vcache = nullptr;
  int head_dim = 128;
  int n_q_local = 0;
  int n_kv_local = 0;
  int block_size = 64;
  // split-K workspace (fp32 partials) + per-tile arrival counters (kept zero between launches)
  float* ws = nullptr;
  float* ws_red = nullptr;  // zero-initialised fp32 tiles for red.add partials (kept zero between launches)
  int* counters = nullptr;
  // debug: globaltimer stamps of the first CTA pair (producer issue / MMA full-wake / epilogue wake)
  unsigned long long* trace = nullptr;
  unsigned long long* span_start = nullptr;  // profiling: atomicMin of CTA start times (globaltimer)
  unsigned long long* span_end = nullptr;    // profiling: atomicMax of CTA end times
  int dbg = 0;  // debug: bit0 skip X loads, bit1 skip W loads, bit2 skip whole-tile epilogue stores (timing experiments only; results invalid)
  // X produced by the still-running predecessor grids (the O projection after the attention
  // kernels): instead of the grid dependency, the TMA producer waits, per k-block kb, for
  // xflag[(kb * 64) / xflag_cols] >= xepoch and once for *xflag2 >= xepoch (if set); the MMA warp
  // does not wait at all and the epilogue keeps the grid dependency (it touches other buffers)
  const unsigned* xflag = nullptr;
  int xflag_cols = 0;
  int xflag_n = 0;  // number of X flags
  const unsigned* xflag2 = nullptr;
  unsigned xepoch = 0;
  // RMSNorm prologue (replaces the rmsnorm kernel before this GEMM): after the grid dependency,
  // the CTAs normalise rows r = blockIdx, blockIdx + grid, ... of norm_h (fp32 [T][norm_H]) into
  // the GEMM's own X (norm_out, bf16 [T][norm_H]: x * rsqrt(mean x^2 + eps) * g, reading O-8), then
  // meet at a grid barrier (monotonic counter: wait for norm_target arrivals) before any X load
  const float* norm_h = nullptr;
  const void* norm_g = nullptr;
  void* norm_out = nullptr;
  int norm_T = 0, norm_H = 0;
  float norm_eps = 0.f;
  unsigned* norm_ctr = nullptr;
  unsigned norm_target = 0;
  // RMSNorm epilogue (EPI_ADD_F32 only; replaces the rmsnorm kernel AFTER this GEMM): once every
  // CTA's residual adds landed (grid barrier on norm_ctr / norm_target), the CTAs normalise rows of
  // out (fp32 [norm_T][norm_H]) into pnorm_out (bf16) with gains pnorm_g and eps norm_eps
  const void* pnorm_g = nullptr;
  void* pnorm_out = nullptr;
  // flag chaining (world 1): every CTA counts itself into *done_ctr after its epilogue's stores /
  // residual adds (the next kernel waits on the count instead of this grid's completion)
  unsigned* done_ctr = nullptr;
  int kbasm = 1;  // MMA issue: a k-block's UMMAs in one asm block (set by launch_gemm)
  int relaxed_rel = 1;  // TMEM-slot releases by relaxed (not release) cluster arrives (set by launch_gemm)
};

struct GemmPlan {
  int M = 0, N = 0, K = 0;
  int bn = 0;          // tokens per tile (multiple of 16, <= 512)
  int n_mma = 1;       // UMMAs per k-step (bn / n_mma <= 256 tokens each)
  int box_rows = 0;    // X TMA box rows (per CTA of the pair: half of UMMA 0's tokens)
  int n0 = 0, n1 = 0;  // tokens of UMMA 0 / 1 (n_mma == 2); uneven (256 + tail) for single-segment plans
  int box_rows2 = 0;   // X box rows of UMMA 1 (n1 / 2) when the split is uneven
  int pm_tiles = 0;    // 256-row tiles (one per CTA pair)
  int m_tiles = 0, n_tiles = 0;  // 128-row tiles (2 * pm_tiles), token tiles
  long long units = 0; // stream-K (pair tile, k-block) units = sk_tiles * K/64
  int ctas = 0;        // persistent grid size in CTA PAIRS
  int tiles = 0;       // pair-tiles (pm_tiles * n_tiles)
  int sk_tiles = 0;    // tiles split stream-K across all pairs (processed first)
  int dp_per_pair = 0; // whole tiles per pair processed after the stream-K part
  int dp_extra = 0;    // pairs [0, dp_extra) take one extra whole tile
  int half_items = 0;  // token-half items after the whole tiles: pair q < half_items runs UMMA (q & 1)'s
                       // tokens of tile tiles - half_items/2 + q/2 (no split-K, no reduction)
  int max_slots = 1;   // stream-K partial slots per tile
  int red_partials = 0;  // split tiles accumulate by red.add into ONE zeroed slot (ws_red)
  int atomic = 0;        // residual-add split tiles red.add every contributor's partial into the output
  int nbuf = 1;        // TMEM accumulator buffers
  int splits = 1, kb_per_split = 0;  // units per CTA (informational)
  int stages = 0;
  size_t smem = 0;
  size_t ws_floats = 0;  // stream-K workspace needed
};

// Workspace convention (ws_cap_floats): slot partials use the lower half, red.add partials the
// upper half, which the caller zeroes once (EpiParams.ws_red = ws + ws_cap_floats / 2).
// Persistent stream-K plan for C[N x M] = X[N x K] * W[M x K]^T on `num_sms` SMs (CTA pairs,
// tcgen05 cta_group::2).  force_pairs > 0 fixes the grid (tests use it to exercise multi-pair
// reductions of one tile).
// atomic_epilogue: the epilogue is a residual add (split tiles reduce with red.add, no reduction pass).
// deterministic: no red.add reductions anywhere (split tiles reduce through partial slots summed
// in slot order by the last contributor; a residual-add epilogue then adds ONE sum per element), so
// a launch's result is bitwise reproducible run to run (slower: DESIGN.md §6).
GemmPlan plan_gemm(int M, int N, int K, int num_sms, size_t ws_cap_floats, int force_pairs = 0,
                   bool atomic_epilogue = false, bool deterministic = false);

// 2D bf16 K-major tensor map with 128B swizzle: rows x cols(=K), box = box_rows x 64.
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_stride_elems, uint32_t box_rows);

// Tensor map over a tile-major, pre-swizzled weight (launch_pack_weight layout): each 16 KB tile
// is read as 32 rows x 512 B (unswizzled box; the bytes are already the SW128 smem image).
bool make_tmap_weight(CUtensorMap* map, const void* w, int M, int K);
// mapW: make_tmap_weight map; mapX: activation [N][K] map (make_tmap_bf16, box rows plan.box_rows).
// mapX2: X map with box rows plan.box_rows2 (uneven split), else ignored (may equal mapX)
cudaError_t launch_gemm(const CUtensorMap& mapW, const CUtensorMap& mapX, const CUtensorMap& mapX2, const GemmPlan& plan,
                        const EpiParams& ep, cudaStream_t stream);

// Debug: prints the globaltimer trace (EpiParams.trace, 4096 u64) of the first CTA pair to stderr.
void dump_gemm_trace(const unsigned long long* trace_dev, const GemmPlan& plan);

// ---------------------------------------------------------------------------
// Layer chain: O-proj -> FFN1 -> FFN2 -> next layer's QKV as ONE persistent launch (gemm_chain.cu).
// Job j+1 reads job j's output through per-128-row-tile flags (flag >= epoch) instead of a kernel
// boundary, so a pair that finishes its share of one GEMM starts the next, the tile quantization
// of one job is filled by the next, and no RMSNorm launch sits between them: a residual-add job's
// tiles are finalised by their last contributor, which writes X = bf16(g * h) for its 128 columns
// and the per-token partial sum of squares; the consuming job's epilogue scales token t by
// rsqrt(sum_parts / H + eps) (RMSNorm is a per-token scale, so it commutes with the GEMM).
constexpr int kChainMaxJobs = 4;
struct ChainJobDev {
  EpiParams ep;                      // mode: EPI_ADD_F32 / EPI_SILU_MUL / EPI_GELU / EPI_QKV_ROPE
  int M = 0, KB = 0;                 // weight rows, k-blocks
  const unsigned* dep_flag = nullptr;  // X k-block kb waits for dep_flag[kb >> dep_shift] >= epoch
  int dep_shift = 0;
  // norm-free input (X = bf16(g * h)): the epilogue scales token t by rsqrt(sum_p ss_in[p][t] * inv_h + eps)
  const float* ss_in = nullptr;      // [ss_parts][ss_ld]; published with dep_flag[0 .. ss_parts)
  int ss_parts = 0;
  float inv_h = 0.f, eps = 0.f;
  // split whole-tile jobs (activation / RoPE epilogues): the need[pt] contributors of a pair tile
  // bulk-reduce-add their partials into scratch slabs (ChainMaps::scr columns slab[pt] * 256 +
  // rank * 128 ...); the last to arrive loads the sum back, adds its own accumulator, runs the
  // epilogue and re-zeroes the slab
  const int* slab = nullptr;         // [pair tiles] slab of a split tile (-1: whole tile)
  int* arrive = nullptr;             // [2 * pair tiles] arrivals / partials reduced (zero between launches)
  int* written = nullptr;
  // residual-add finalisation (per 128-row tile; the last of need[pair tile] contributors):
  // fin_xa[t][col] = bf16(fin_g[col] * h[t][col]), fin_ss[tile][t] = sum_col h^2, flag_out[tile] = epoch
  int* fin_cnt = nullptr;            // [2 * pair tiles], zero between launches
  const int* fin_need = nullptr;     // [pair tiles]
  const void* fin_g = nullptr;       // bf16 [M]
  void* fin_xa = nullptr;            // bf16 [tokens][M]
  float* fin_ss = nullptr;           // [M / 128][ss_ld]
  unsigned* flag_out = nullptr;      // whole-tile jobs: set after the tile's epilogue; split: after finalisation
};
struct ChainLaunch {
  ChainJobDev job[kChainMaxJobs];
  int njobs = 0;
  const int* segs = nullptr;         // device: 4 ints per segment (job, pair tile, kb0, kb1)
  const int* seg_off = nullptr;      // device: [pairs + 1]
  int pairs = 0;
  int N = 0, bn = 0, n_mma = 1, stages = 0, nbuf = 1;
  int ss_ld = 0;                     // row stride of the ss arrays (max tokens)
  float* scr = nullptr;              // split-tile scratch base (row stride scr_ld floats), zero between launches
  int scr_ld = 0;
  unsigned epoch = 0;
  size_t smem = 0;
  uint32_t tmem_cols = 0, ring_bytes = 0;
  unsigned long long* span_start = nullptr;
  unsigned long long* span_end = nullptr;
  // debug timeline (SARATHI_CHAIN_TRACE): [pairs][kChainTraceSegs][8] globaltimer stamps of the
  // leader CTA: mma start / first stage / last commit, epilogue wake / published, producer dep-wait ns
  unsigned long long* trace = nullptr;
  int kbasm = 1;     // a k-block's UMMAs from one asm block (set by launch_chain; SARATHI_GEMM_KBASM=0: per UMMA)
  int relaxed = 1;   // relaxed cluster arrives for TMEM-slot releases (SARATHI_GEMM_RELAXED=0: release)
};
constexpr int kChainTraceSegs = 16;
struct ChainMaps {
  CUtensorMap w[kChainMaxJobs];      // make_tmap_weight maps
  CUtensorMap x[kChainMaxJobs];      // activation maps, box rows bn / n_mma / 2
  CUtensorMap hred;                  // fp32 residual h [T][H], box 32 columns x 16 tokens (TMA reduce-add)
  CUtensorMap scr;                   // fp32 split-tile scratch [T][slabs * 256], same box
};
// fp32 [rows][cols] map with a 32-column x 16-row box, no swizzle (bulk reduce-add target).
bool make_tmap_f32_red(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems);
// Token tiling / ring of a chain over N tokens (N <= 512: one token tile).  Fills bn, n_mma,
// stages, nbuf, smem, tmem_cols, ring_bytes; returns false if N needs more than one token tile.
bool plan_chain_tiling(int N, ChainLaunch* cl);
cudaError_t launch_chain(const ChainMaps& maps, const ChainLaunch& cl, int ffn_mode, cudaStream_t stream);

}  // namespace sarathi

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
  int max_slots = 1;   // stream-K partial slots per tile
  int red_partials = 0;  // split tiles accumulate by red.add into ONE zeroed slot (ws_red)
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
GemmPlan plan_gemm(int M, int N, int K, int num_sms, size_t ws_cap_floats, int force_pairs = 0,
                   bool atomic_epilogue = false);

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

}  // namespace sarathi

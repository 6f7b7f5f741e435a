// Host-visible declarations of the non-GEMM kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda.h>

namespace sarathi {

struct DecodeAttnArgs {
  const __nv_bfloat16* q = nullptr;  // [T][q_ld]; decode j reads row q_row0 + j
  int q_ld = 0;
  int q_row0 = 0;
  const void* kcache = nullptr;  // bf16 [num_blocks][n_kv_local][block_size][head_dim]
  const void* vcache = nullptr;
  const int* block_tables = nullptr;  // [d][max_blocks]
  const int* ctx = nullptr;           // [d] keys to attend (= position + 1)
  int max_blocks = 0;
  int d = 0;
  int n_q_local = 0, n_kv_local = 0, head_dim = 128, block_size = 64;
  float scale = 0.f;
  int splits = 1, blocks_per_split = 1, stages = 2;
  float* part_o = nullptr;    // [d][n_q_local][splits][head_dim]
  float* part_lse = nullptr;  // [d][n_q_local][splits]
  __nv_bfloat16* out = nullptr;  // [T][out_ld]; row q_row0 + j
  int out_ld = 0;
  int dbg = 0;  // timing experiments only: bit0 = consumers skip the math (pure K/V streaming)
  // 0: launched with programmatic dependent launch (CTAs become resident while the QKV GEMM
  // drains).  1: plain launch, so a concurrently pending prefill-attention grid on the
  // high-priority stream is dispatched first when the GEMM completes.
  int no_pdl = 0;
  // 1: this launch directly follows the chunk's prefill attention in the same stream (the
  // "attention chain"): the prefill grid waited for the QKV GEMM before triggering this launch,
  // so q / K / V are complete when the CTAs start; the grid's last CTA instead waits for the
  // prefill grid at its END, so the O projection after it (PDL) sees both attention outputs.
  int wait_at_end = 0;
  // profiling (sarathi_op_kernel_times): min CTA start / max CTA end, globaltimer ns, or null
  unsigned long long* span_start = nullptr;
  unsigned long long* span_end = nullptr;
  // per-KV-head completion (splits == 1): the d-th CTA of KV head g to finish its output rows sets
  // head_flag[g] = epoch (release), so the O projection can start on finished heads inside this
  // grid's last wave (GEMM EpiParams::xflag); head_cnt zero between launches
  unsigned* head_flag = nullptr;
  int* head_cnt = nullptr;
  unsigned epoch = 0;
};

struct PrefillAttnArgs {
  const __nv_bfloat16* q = nullptr;  // [T][q_ld], chunk rows q_row0 .. q_row0+p-1
  int q_ld = 0;
  int q_row0 = 0;
  const void* kcache = nullptr;
  const void* vcache = nullptr;
  const int* block_table = nullptr;  // [max_blocks] of the prefill request
  int start = 0;  // s: tokens cached before the chunk
  int p = 0;      // chunk tokens
  int n_q_local = 0, n_kv_local = 0, head_dim = 128, block_size = 64;
  float scale = 0.f;
  __nv_bfloat16* out = nullptr;
  int out_ld = 0;
  unsigned long long* trace = nullptr;  // debug: globaltimer stamps of CTA (0,0) (tcgen05 kernel)
  int pdl = 0;  // launch with programmatic dependent launch (attention chain; tcgen05 kernel)
  // key split (tcgen05 kernel): each (q-tile, head) pair's key tiles are divided into ksplit
  // contiguous ranges, one CTA each; ranges write unnormalised fp32 O + (m, l) partials and the last
  // CTA of the pair to finish merges them (flash-decoding style) into out.  The host keeps ksplit
  // <= the key-tile count of the first q-tile, so no range is empty.
  int ksplit = 1;
  float* part_o = nullptr;   // [pairs][ksplit][128 rows][head_dim]
  float* part_ml = nullptr;  // [pairs][ksplit][128 rows][2] (running max in log2 units, row sum)
  int* counters = nullptr;   // [pairs], zero between launches (the merging CTA re-zeroes)
  unsigned long long* span_start = nullptr;  // profiling, as DecodeAttnArgs (tcgen05 kernel)
  unsigned long long* span_end = nullptr;
  // grid completion (tcgen05 kernel): the last CTA to finish sets done_flag = epoch (release)
  unsigned* done_flag = nullptr;
  int* done_cnt = nullptr;
  unsigned epoch = 0;
  int mma8 = 1;  // issue S = QK^T / O += PV as 8 UMMAs in one asm block (SARATHI_ATTN_MMA8=0: one asm per UMMA)
};

size_t decode_smem_bytes(int head_dim, int block_size, int stages, int G);
// TMA map over one layer's K or V pool viewed as [num_blocks * n_kv_local * block_size][head_dim].
bool make_tmap_kv(CUtensorMap* map, const void* pool, long long rows, int head_dim, int block_size);
cudaError_t launch_decode_attention(const DecodeAttnArgs& a, const CUtensorMap& kmap, const CUtensorMap& vmap,
                                    cudaStream_t st);
// Chunked-prefill attention.  With the TMA maps (q: [Tmax][q_ld] box 128 x 64; K/V: make_tmap_kv) and
// block_size in {16, 32, 64, 128} it runs the tcgen05 kernel, otherwise the mma.sync kernel.
cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, const CUtensorMap* qmap, const CUtensorMap* kmap,
                                     const CUtensorMap* vmap, cudaStream_t st);

// TP partials to add into the residual before a norm (Megatron row-parallel O / down, PAPER.md L249
// §2.3).  world == 0: nothing.  world == 1: p[0] holds the already all-reduced sum (NCCL path).
// world > 1: the one-shot all-reduce fused into the consumer — p[r] is rank r's bf16 partial (peer
// memory: the same device in a local group, CUDA-IPC mapped over NVLink across processes), summed
// in rank order in fp32 (identical on every rank); when ready != nullptr the kernel first waits until
// ready[r] >= epoch for every rank r (each rank's signal after its GEMM; ld.acquire.sys).
struct PeerSum {
  const __nv_bfloat16* p[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int world = 0;
  const unsigned int* ready = nullptr;
  unsigned int epoch = 0;
  // NVLS: multicast address of the partial buffer; the sum over ranks is ONE
  // multimem.ld_reduce.add.acc::f32 per 4 bf16 (reduced in the NVSwitch) instead of world loads
  const __nv_bfloat16* mm = nullptr;
};

// h[t][:] = float(E[tok[t]][:])
cudaError_t launch_embedding(const int* tok, const __nv_bfloat16* E, float* h, int T, int H, cudaStream_t st);

// Flag chaining of the rmsnorm kernel (world 1): instead of the grid dependency on the preceding
// residual-add GEMM it waits until *wait_ctr >= wait_target (that GEMM's CTAs count themselves in
// after their residual adds), and every CTA counts itself into *done_ctr after its stores (the next
// GEMM's TMA producer waits on that instead of this grid's completion).  Monotonic counters.
struct NormFlags {
  const unsigned* wait_ctr = nullptr;
  unsigned wait_target = 0;
  unsigned* done_ctr = nullptr;
};

// out[r][:] = bf16(RMSNorm(h[row(r)]) * g); row(r) = rows ? rows[r] : r.
// With TP partials (PeerSum world >= 1): h[row] += sum of the partials' row first and h is updated.
cudaError_t launch_rmsnorm(float* h, const PeerSum& add, const __nv_bfloat16* g, __nv_bfloat16* out,
                           const int* rows, int R, int H, float eps, cudaStream_t st,
                           unsigned long long* span_start = nullptr, unsigned long long* span_end = nullptr,
                           const NormFlags& flags = NormFlags());
inline cudaError_t launch_rmsnorm(float* h, const __nv_bfloat16* add, const __nv_bfloat16* g, __nv_bfloat16* out,
                                  const int* rows, int R, int H, float eps, cudaStream_t st,
                                  unsigned long long* span_start = nullptr, unsigned long long* span_end = nullptr) {
  PeerSum ps;
  ps.world = add ? 1 : 0;
  ps.p[0] = add;
  return launch_rmsnorm(h, ps, g, out, rows, R, H, eps, st, span_start, span_end);
}

// h[t][:] += sum of the partials (PeerSum, world >= 1), no norm (last layer under TP before the
// final norm)
cudaError_t launch_residual_add(float* h, const PeerSum& add, int T, int H, cudaStream_t st);

// logits[r][rank*Vl + c] = gathered[rank][r][c]  (vocab-parallel all-gather layout -> [R][V])
cudaError_t launch_vocab_permute(const float* gathered, float* logits, int world, int R, int Vl, int V,
                                 cudaStream_t st);

// Device weight generator (same counter-based spec as synth/__init__.py, independent code).
// dst[r][c] = bf16_rne( f32(2*u24 - (2^24-1)) * scale[r] ), u24 = splitmix64(seed ^ (tau[r] << 40 | base[r] + c)) >> 40
// packed != 0: write the tile-major GEMM layout (see packed_weight_index); dst must hold
// ceil(rows/128)*128 rows (padding rows zeroed by the caller).
cudaError_t launch_weightgen(__nv_bfloat16* dst, int rows, int cols, const int* tau, const float* scale,
                             const long long* base, unsigned long long seed, int packed, cudaStream_t st);
// Row-major [rows][cols] -> tile-major, SW128-pre-swizzled GEMM layout: element (r, c) at
// ((r/128)*(cols/64) + c/64)*8192 + (r%128)*64 + (((c%64)/8) ^ (r%8))*8 + c%8.
cudaError_t launch_pack_weight(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int cols, cudaStream_t st);
inline size_t packed_weight_index(int r, int c, int cols) {
  const int rr = r & 127, j = (c & 63) >> 3;
  return ((static_cast<size_t>(r >> 7) * (cols >> 6) + (c >> 6)) << 13) + (rr << 6) + ((j ^ (rr & 7)) << 3) + (c & 7);
}
// dst[i] = bf16_rne( 1.0f + f32(v) * f32(0.1/2^24) )  over flat indices [base, base+n)
cudaError_t launch_gaingen(__nv_bfloat16* dst, int n, int tau, long long base, unsigned long long seed,
                           cudaStream_t st);

}  // namespace sarathi

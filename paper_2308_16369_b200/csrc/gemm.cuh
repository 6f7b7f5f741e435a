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
  EPI_SILU_MUL = 3,    // gate/up interleaved in 64-row blocks: out[t, f] = bf16(silu(g) * u)
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
  const float* rope_cos = nullptr;  // [max_pos][head_dim/2]
  const float* rope_sin = nullptr;
  void* kcache = nullptr;  // bf16 [num_blocks][n_kv_local][block_size][head_dim]
  void* vcache = nullptr;
  int head_dim = 128;
  int n_q_local = 0;
  int n_kv_local = 0;
  int block_size = 64;
  // split-K workspace (fp32 partials) + per-tile arrival counters (kept zero between launches)
  float* ws = nullptr;
  int* counters = nullptr;
};

struct GemmPlan {
  int M = 0, N = 0, K = 0;
  int bn = 0;          // tokens per CTA tile (multiple of 16, <= 256)
  int m_tiles = 0, n_tiles = 0;
  int splits = 1, kb_per_split = 0;
  int stages = 0;
  size_t smem = 0;
  size_t ws_floats = 0;  // workspace needed (splits > 1)
};

// Choose tile / split-K for C[N x M] = X[N x K] * W[M x K]^T on `num_sms` SMs.
GemmPlan plan_gemm(int M, int N, int K, int num_sms, size_t ws_cap_floats, int force_splits = 0);

// 2D bf16 K-major tensor map with 128B swizzle: rows x cols(=K), box = box_rows x 64.
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_stride_elems, uint32_t box_rows);

cudaError_t launch_gemm(const CUtensorMap& mapW, const CUtensorMap& mapX, const GemmPlan& plan,
                        const EpiParams& ep, cudaStream_t stream);

}  // namespace sarathi

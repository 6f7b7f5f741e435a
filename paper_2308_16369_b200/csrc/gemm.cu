// tcgen05 / TMEM / TMA bf16 GEMM for the hybrid-batch linears (preproj, postproj, ffn_ln1,
// ffn_ln2 and the LM head; PAPER.md L214-221 Table table:tensor:shapes, §2.1).
//
// Decode-maximal batching fuses all p + d tokens of a hybrid batch into ONE matmul per linear so
// every weight byte is fetched once for both kinds of token (§4.3).  With
// T = p + d <= 512 tokens per batch, the natural sm_100a mapping is "swap-AB":
//   D[m, t] = sum_k W[m, k] * X[t, k]       (UMMA M = 128 weight rows, N = bn tokens, K = 16/instr)
// so each CTA streams a 128-row weight slab exactly once from HBM while the (small, L2-resident)
// token matrix is re-read from L2.  Pipeline per CTA (192 threads, 1 CTA / SM):
//   warp 0      TMA producer: W tile [128 x 64] (evict_first) + X tile [bn x 64] (evict_last),
//               128B swizzle, into an S-stage smem ring (full/empty mbarriers)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; tcgen05.commit frees stages
//   warps 2..5  epilogue: tcgen05.ld TMEM -> regs -> (split-K partial | smem tile) -> fused op
// Split-K (grid.z) writes fp32 partials; the last-arriving CTA of a tile (atomic counter) reduces
// them in split order (deterministic) and runs the epilogue.
#include "common.cuh"
#include "gemm.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace sarathi {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kStilePitch = 132;             // fp32 staging row pitch (128 + 4 pad)
constexpr int kThreads = 192;

struct KParams {
  int M, N, KB, bn, m_tiles, n_tiles, splits, kb_per_split, stages;
  uint32_t tmem_cols;
  uint32_t smem_main;  // bytes of ring / staging region
};

SARATHI_DEVICE float silu_f(float x) { return x / (1.0f + __expf(-x)); }
SARATHI_DEVICE float gelu_tanh_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}

__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap mapW,
                        const __grid_constant__ CUtensorMap mapX, const KParams p,
                        const EpiParams ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t b_bytes = static_cast<uint32_t>(p.bn) * kBK * 2;
  const uint32_t stage_bytes = kABytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.smem_main);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint32_t* holder = reinterpret_cast<uint32_t*>(tfull + 1);
  __shared__ int s_last;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int mt = blockIdx.x, nt = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int nk = min(p.kb_per_split, p.KB - kb0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapW);
    tma_prefetch_desc(&mapX);
  }
  if (warp == 1) tmem_alloc(holder, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      for (int i = 0; i < nk; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (i / p.stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* a = smem + static_cast<size_t>(s) * stage_bytes;
        uint8_t* b = a + kABytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(a, &mapW, &full[s], kc, mt * kBM, pol_w);
        tma_load_2d(b, &mapX, &full[s], kc, nt * p.bn, pol_x);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (lane 0 issues and commits) ----------------
    const uint32_t idesc = make_idesc_bf16_f32(kBM, p.bn);
    for (int i = 0; i < nk; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (i / p.stages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
        const uint32_t b = a + kABytes;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          umma_f16_ss(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc,
                      (i | k) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        if (i == nk - 1) umma_commit(tfull);
      }
      __syncwarp();
    }
  } else {
    // ---------------- Epilogue (warps 2..5) ----------------
    const int et = threadIdx.x - 64;             // 0..127
    const uint32_t quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int r = static_cast<int>(quarter * 32 + lane);  // accumulator row (weight row in tile)
    float* stile = reinterpret_cast<float*>(smem);        // [bn][kStilePitch] fp32, reuses ring
    mbar_wait(tfull, 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((quarter * 32u) << 16);

    bool do_epilogue = true;
    if (p.splits > 1) {
      const size_t tile_elems = static_cast<size_t>(p.bn) * kBM;
      float* wsp = ep.ws + (static_cast<size_t>(split * p.m_tiles + mt) * p.n_tiles + nt) * tile_elems;
      for (int c0 = 0; c0 < p.bn; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcg(wsp + static_cast<size_t>(c0 + j) * kBM + r, __uint_as_float(v[j]));
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (et == 0) {
        int* ctr = ep.counters + mt * p.n_tiles + nt;
        const int old = atomicAdd(ctr, 1);
        s_last = (old == p.splits - 1);
        if (s_last) *ctr = 0;  // re-arm for the next launch
      }
      named_bar_sync(1, 128);
      do_epilogue = s_last != 0;
      if (do_epilogue) {
        __threadfence();
        const float* base = ep.ws + (static_cast<size_t>(mt) * p.n_tiles + nt) * tile_elems;
        const size_t split_stride = static_cast<size_t>(p.m_tiles) * p.n_tiles * tile_elems;
        for (int c = 0; c < p.bn; ++c) {
          float acc = 0.f;
          for (int s = 0; s < p.splits; ++s)
            acc += __ldcg(base + s * split_stride + static_cast<size_t>(c) * kBM + r);
          stile[c * kStilePitch + r] = acc;
        }
      }
    } else {
      for (int c0 = 0; c0 < p.bn; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) stile[(c0 + j) * kStilePitch + r] = __uint_as_float(v[j]);
      }
    }

    if (do_epilogue) {
      named_bar_sync(1, 128);
      const int ew = et >> 5;
      const int tvalid = min(p.bn, p.N - nt * p.bn);
      const int m0 = mt * kBM;
      const int f = static_cast<int>(lane) * 4;
      switch (ep.mode) {
        case EPI_STORE_BF16:
        case EPI_GELU: {
          __nv_bfloat16* out = static_cast<__nv_bfloat16*>(ep.out);
          const bool gelu = ep.mode == EPI_GELU;
          for (int t = ew; t < tvalid; t += 4) {
            const float4 v = *reinterpret_cast<const float4*>(stile + t * kStilePitch + f);
            float x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
            if (gelu) { x0 = gelu_tanh_f(x0); x1 = gelu_tanh_f(x1); x2 = gelu_tanh_f(x2); x3 = gelu_tanh_f(x3); }
            __nv_bfloat16* dst = out + static_cast<long long>(nt * p.bn + t) * ep.ldo + m0 + f;
            if (m0 + f + 3 < p.M) {
              uint2 pk = make_uint2(pack_bf16x2(x0, x1), pack_bf16x2(x2, x3));
              *reinterpret_cast<uint2*>(dst) = pk;
            } else {
              const float xs[4] = {x0, x1, x2, x3};
              for (int j = 0; j < 4; ++j)
                if (m0 + f + j < p.M) dst[j] = __float2bfloat16_rn(xs[j]);
            }
          }
          break;
        }
        case EPI_STORE_F32:
        case EPI_ADD_F32: {
          float* out = static_cast<float*>(ep.out);
          const bool add = ep.mode == EPI_ADD_F32;
          for (int t = ew; t < tvalid; t += 4) {
            float4 v = *reinterpret_cast<const float4*>(stile + t * kStilePitch + f);
            float* dst = out + static_cast<long long>(nt * p.bn + t) * ep.ldo + m0 + f;
            if (m0 + f + 3 < p.M) {
              if (add) {
                const float4 o = *reinterpret_cast<const float4*>(dst);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(dst) = v;
            } else {
              const float xs[4] = {v.x, v.y, v.z, v.w};
              for (int j = 0; j < 4; ++j)
                if (m0 + f + j < p.M) dst[j] = add ? dst[j] + xs[j] : xs[j];
            }
          }
          break;
        }
        case EPI_SILU_MUL: {
          // rows [0,64) of the tile are gate features, [64,128) the matching up features.
          __nv_bfloat16* out = static_cast<__nv_bfloat16*>(ep.out);
          const int fo = static_cast<int>(lane) * 2;
          for (int t = ew; t < tvalid; t += 4) {
            const float* srow = stile + t * kStilePitch;
            const float2 g = *reinterpret_cast<const float2*>(srow + fo);
            const float2 u = *reinterpret_cast<const float2*>(srow + 64 + fo);
            __nv_bfloat16* dst = out + static_cast<long long>(nt * p.bn + t) * ep.ldo + mt * 64 + fo;
            *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(silu_f(g.x) * u.x, silu_f(g.y) * u.y);
          }
          break;
        }
        case EPI_QKV_ROPE: {
          const int hd = ep.head_dim, half = hd >> 1;
          __nv_bfloat16* qout = static_cast<__nv_bfloat16*>(ep.out);
          __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(ep.kcache);
          __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(ep.vcache);
          const int pr = static_cast<int>(lane) * 2;   // first of this lane's two pairs
          const int hh = pr / half, d = pr % half;     // head within tile, dim within half
          const int f1 = hh * hd + d;
          const int gm = m0 + f1;                      // global feature of x1
          if (gm < p.M) {
            const int gh = gm / hd;                    // global head index in [q | k | v]
            for (int t = ew; t < tvalid; t += 4) {
              const float* srow = stile + t * kStilePitch;
              const int gt = nt * p.bn + t;
              float2 x1 = *reinterpret_cast<const float2*>(srow + f1);
              float2 x2 = *reinterpret_cast<const float2*>(srow + f1 + half);
              if (gh < ep.n_q_local + ep.n_kv_local) {
                const int ps = ep.pos[gt];
                const float2 c = *reinterpret_cast<const float2*>(ep.rope_cos + static_cast<size_t>(ps) * half + d);
                const float2 s = *reinterpret_cast<const float2*>(ep.rope_sin + static_cast<size_t>(ps) * half + d);
                const float2 y1 = make_float2(x1.x * c.x - x2.x * s.x, x1.y * c.y - x2.y * s.y);
                const float2 y2 = make_float2(x2.x * c.x + x1.x * s.x, x2.y * c.y + x1.y * s.y);
                x1 = y1;
                x2 = y2;
              }
              if (gh < ep.n_q_local) {
                __nv_bfloat16* dst = qout + static_cast<long long>(gt) * ep.ldo + gh * hd + d;
                *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(x1.x, x1.y);
                *reinterpret_cast<uint32_t*>(dst + half) = pack_bf16x2(x2.x, x2.y);
              } else {
                const bool isk = gh < ep.n_q_local + ep.n_kv_local;
                const int kvh = isk ? gh - ep.n_q_local : gh - ep.n_q_local - ep.n_kv_local;
                const int sl = ep.slot[gt];
                const size_t row = (static_cast<size_t>(sl / ep.block_size) * ep.n_kv_local + kvh) * ep.block_size +
                                   sl % ep.block_size;
                __nv_bfloat16* dst = (isk ? kc : vc) + row * hd + d;
                *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(x1.x, x1.y);
                *reinterpret_cast<uint32_t*>(dst + half) = pack_bf16x2(x2.x, x2.y);
              }
            }
          }
          break;
        }
        default:
          break;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  }
  return fn;
}

uint32_t pow2_cols(int n) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(n)) c <<= 1;
  return c;
}

}  // namespace

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_stride_elems, uint32_t box_rows) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

GemmPlan plan_gemm(int M, int N, int K, int num_sms, size_t ws_cap_floats, int force_splits) {
  GemmPlan pl;
  pl.M = M;
  pl.N = N;
  pl.K = K;
  const int KB = K / kBK;
  pl.n_tiles = (N + 255) / 256;
  const int per = (N + pl.n_tiles - 1) / pl.n_tiles;
  pl.bn = std::max(16, (per + 15) / 16 * 16);
  pl.m_tiles = (M + kBM - 1) / kBM;
  const size_t tile_elems = static_cast<size_t>(pl.bn) * kBM;

  double best = 1e300;
  int best_s = 1, best_kbps = KB;
  const int smax = std::min(32, KB);
  for (int s = 1; s <= smax; ++s) {
    const int kbps = (KB + s - 1) / s;
    const int s_eff = (KB + kbps - 1) / kbps;
    if (s_eff != s) continue;
    if (force_splits > 0 && s != force_splits) continue;
    const size_t ws_need = s > 1 ? static_cast<size_t>(s) * pl.m_tiles * pl.n_tiles * tile_elems : 0;
    if (ws_need > ws_cap_floats) continue;
    const int ctas = pl.m_tiles * pl.n_tiles * s;
    const int waves = (ctas + num_sms - 1) / num_sms;
    const int active = std::min(ctas, num_sms);
    // cycles per k-block per CTA: MMA (2*bn) vs this CTA's share of HBM weight streaming
    const double t_kb = std::max(2.0 * pl.bn, kABytes * static_cast<double>(active) / 3400.0) + 64.0;
    double est = waves * (kbps * t_kb + 1500.0);
    if (s > 1) est += 800.0 + s * pl.bn * 4.0;  // partial write + last-CTA reduction
    if (est < best * 0.98) {
      best = est;
      best_s = s;
      best_kbps = kbps;
    }
  }
  pl.splits = best_s;
  pl.kb_per_split = best_kbps;
  pl.ws_floats = pl.splits > 1 ? static_cast<size_t>(pl.splits) * pl.m_tiles * pl.n_tiles * tile_elems : 0;
  const size_t stage = kABytes + static_cast<size_t>(pl.bn) * kBK * 2;
  const size_t budget = 224 * 1024;
  int stages = static_cast<int>(std::min<size_t>(8, (budget - 2048) / stage));
  stages = std::max(2, std::min(stages, std::max(2, pl.kb_per_split)));
  pl.stages = stages;
  const size_t main = std::max(stages * stage, static_cast<size_t>(pl.bn) * kStilePitch * 4);
  pl.smem = main + 1024 + 256;
  return pl;
}

cudaError_t launch_gemm(const CUtensorMap& mapW, const CUtensorMap& mapX, const GemmPlan& pl,
                        const EpiParams& ep, cudaStream_t stream) {
  static size_t configured = 0;
  if (pl.smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(std::max<size_t>(pl.smem, 200 * 1024)));
    if (e != cudaSuccess) return e;
    configured = std::max<size_t>(pl.smem, 200 * 1024);
  }
  KParams kp;
  kp.M = pl.M;
  kp.N = pl.N;
  kp.KB = pl.K / kBK;
  kp.bn = pl.bn;
  kp.m_tiles = pl.m_tiles;
  kp.n_tiles = pl.n_tiles;
  kp.splits = pl.splits;
  kp.kb_per_split = pl.kb_per_split;
  kp.stages = pl.stages;
  kp.tmem_cols = pow2_cols(pl.bn);
  const size_t stage = kABytes + static_cast<size_t>(pl.bn) * kBK * 2;
  kp.smem_main = static_cast<uint32_t>(std::max(pl.stages * stage, static_cast<size_t>(pl.bn) * kStilePitch * 4));
  dim3 grid(pl.m_tiles, pl.n_tiles, pl.splits);
  gemm_bf16_tc_kernel<<<grid, kThreads, pl.smem, stream>>>(mapW, mapX, kp, ep);
  return cudaGetLastError();
}

}  // namespace sarathi

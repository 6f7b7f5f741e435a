// Microbenchmark: the GEMM's real fused epilogues (gemm_epi.cuh epi_emit) on their own, in the GEMM's
// launch shape (one CTA per SM, 320 threads, warps 2..9 drain TMEM lane quarters, two warps per
// quarter, one 16-token chunk in flight), over T tokens of one 128-row tile per CTA.  Separates the
// epilogue's own cost from its environment inside the GEMM (DESIGN.md §6 / §10).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2308_16369_b200/csrc \
//        -o tools/epi_bench tools/epi_bench.cu
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_epi.cuh"

using namespace sarathi;

namespace sarathi {
namespace {
// (experiment, measured no faster: 6.85 vs 7.10 us) Two 16-token chunks (c0, c0 + 16) of the fused QKV epilogue in one pass: one TMEM wait, the
// RoPE of both chunks as independent chains (their shuffles / recurrences / sincos overlap), one
// 2 KB bf16 transpose (32 tokens x 32 rows) and four 16-B store passes.  Same results as two
// epi_emit<EPI_QKV_ROPE> calls (identical per-token arithmetic).
SARATHI_DEVICE void epi_qkv32(const int M, const int bn, const EpiParams& ep, float (&v)[32], uint32_t q, uint32_t lane,
                              int mt, int nt, int c0, int tvalid, float* sbuf, const int* s_pos, const int* s_slot,
                              const int* s_consec, const QkvLane& ql) {
  const int row0 = mt * kBM + static_cast<int>(q) * 32;
  const long long tb = static_cast<long long>(nt) * bn + c0;
  const int nv = min(32, tvalid - c0);
  uint16_t* sb = reinterpret_cast<uint16_t*>(sbuf);
  const int half = ep.head_dim >> 1;
  const bool lo = lane < 16;
  if (ql.rope) {
    const float cd = ql.cd, sd = ql.sd;
    float cr[2], sr[2];
    bool cons[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int cc = c0 + 16 * hh;
      cons[hh] = cc < tvalid && s_consec[cc >> 4] != 0;
      cr[hh] = 1.f;
      sr[hh] = 0.f;
      if (cons[hh]) rope_cos_sin(s_pos[cc], ql.th_hi, ql.th_lo, cr[hh], sr[hh]);
    }
    float xp[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) xp[j] = __shfl_xor_sync(0xffffffffu, v[j], 16);  // rotate-half partners
#pragma unroll
    for (int j8 = 0; j8 < 2; ++j8) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j0 = 16 * hh + 8 * j8;
        float c[8], sn[8];
        if (cons[hh]) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            c[j] = cr[hh];
            sn[j] = sr[hh];
            const float cn = fmaf(cr[hh], cd, -sr[hh] * sd);
            sr[hh] = fmaf(sr[hh], cd, cr[hh] * sd);
            cr[hh] = cn;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) rope_cos_sin(s_pos[min(c0 + j0 + j, tvalid - 1)], ql.th_hi, ql.th_lo, c[j], sn[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float y = lo ? v[j0 + j] * c[j] - xp[j0 + j] * sn[j] : v[j0 + j] * c[j] + xp[j0 + j] * sn[j];
          sb[(j0 + j) * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(y));
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) sb[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(v[j]));
  }
  __syncwarp();
  if (row0 < M) {
    const int hd_shift = ep.head_dim == 128 ? 7 : 6;
    const bool isq = ql.gh < ep.n_q_local;
    const int kvh = isq ? 0 : (ql.rope ? ql.gh - ep.n_q_local : ql.gh - ep.n_q_local - ep.n_kv_local);
    __nv_bfloat16* cache = static_cast<__nv_bfloat16*>(ql.rope ? ep.kcache : ep.vcache);
    const int g = static_cast<int>(lane & 3);
    const int d = (g < 2 ? 0 : half) + 16 * ql.jw + (g & 1) * 8;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int tok = pass * 8 + static_cast<int>(lane >> 2);
      if (tok >= nv) continue;
      __nv_bfloat16* dst =
          isq ? static_cast<__nv_bfloat16*>(ep.out) + (tb + tok) * ep.ldo + (ql.gh << hd_shift) + d
              : cache + (static_cast<size_t>(s_slot[c0 + tok] + kvh * ep.block_size) << hd_shift) + d;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(sb + tok * 32 + g * 8);
    }
  }
  __syncwarp();
}

}  // namespace
}  // namespace sarathi

template <int MODE, bool DBG = false, int VAR = 0>
__global__ void __launch_bounds__(320, 1) epi_kernel(EpiParams ep, int M, int T, unsigned long long* out) {
  __shared__ uint32_t holder;
  __shared__ __align__(16) float stage[8][kStageFloats];
  __shared__ int s_pos[512], s_slot[512], s_consec[32];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) tmem_alloc(&holder, 512);
  const int mt = blockIdx.x;  // this CTA's 128-row tile
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    s_pos[t] = __ldg(ep.pos + t);
    const int sl = __ldg(ep.slot + t);
    s_slot[t] = (sl / ep.block_size) * ep.n_kv_local * ep.block_size + sl % ep.block_size;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < (T + 15) / 16) {
    const int c0 = threadIdx.x * 16, n = min(16, T - c0);
    int ok = 1;
    for (int j = 1; j < n; ++j) ok &= s_pos[c0 + j] == s_pos[c0] + j;
    s_consec[threadIdx.x] = ok;
  }
  __syncthreads();
  const uint32_t tmem = holder;
  const unsigned long long t0 = globaltimer_ns();
  if (warp >= 2) {
    const uint32_t quarter = warp & 3, eh = (warp - 2) >> 2;
    const uint32_t trow = tmem + ((quarter * 32u) << 16);
    QkvLane ql{};
    if (MODE == EPI_QKV_ROPE) ql = qkv_lane(ep, mt, quarter, lane);
    const int nchunks = (T + 15) / 16;
    if (VAR == 1) {  // two chunks per TMEM wait (chunk pairs 2(eh + 2i), +1), two epi_emit calls
      for (int c2 = 2 * eh; c2 < nchunks; c2 += 4) {
        uint32_t ra[16], rb[16];
        tmem_ld_32x32b_x16(trow + (c2 % 32) * 16, ra);
        tmem_ld_32x32b_x16(trow + ((c2 + 1) % 32) * 16, rb);
        tmem_ld_wait_regs(ra);
        regs_fence(rb);
        float va[16], vb[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          va[j] = __uint_as_float(ra[j]) * 1e-30f + 0.01f * j;
          vb[j] = __uint_as_float(rb[j]) * 1e-30f + 0.01f * j;
        }
        epi_emit<MODE, DBG>(M, 512, ep, va, quarter, lane, mt, 0, c2 * 16, T, stage[warp - 2], s_pos, s_slot, s_consec, ql);
        if (c2 + 1 < nchunks)
          epi_emit<MODE, DBG>(M, 512, ep, vb, quarter, lane, mt, 0, (c2 + 1) * 16, T, stage[warp - 2], s_pos, s_slot, s_consec, ql);
      }
    } else if (VAR == 2) {  // 32-token QKV emitter
      for (int c2 = 2 * eh; c2 < nchunks; c2 += 4) {
        uint32_t ra[16], rb[16];
        tmem_ld_32x32b_x16(trow + (c2 % 32) * 16, ra);
        tmem_ld_32x32b_x16(trow + ((c2 + 1) % 32) * 16, rb);
        tmem_ld_wait_regs(ra);
        regs_fence(rb);
        float v[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[j] = __uint_as_float(ra[j]) * 1e-30f + 0.01f * j;
          v[16 + j] = __uint_as_float(rb[j]) * 1e-30f + 0.01f * j;
        }
        epi_qkv32(M, 512, ep, v, quarter, lane, mt, 0, c2 * 16, T, stage[warp - 2], s_pos, s_slot, s_consec, ql);
      }
    } else
    for (int ch = eh; ch < nchunks; ch += 2) {
      uint32_t raw[16];
      tmem_ld_32x32b_x16(trow + (ch % 32) * 16, raw);
      tmem_ld_wait_regs(raw);
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]) * 1e-30f + 0.01f * j;  // TMEM garbage -> finite
      epi_emit<MODE, DBG>(M, 512, ep, v, quarter, lane, mt, 0, ch * 16, T, stage[warp - 2], s_pos, s_slot, s_consec, ql);
    }
  }
  __syncthreads();
  if (threadIdx.x == 64) out[blockIdx.x] = globaltimer_ns() - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE, bool DBG = false, int VAR = 0>
void run(const char* name, EpiParams ep, int M, int T, int ctas) {
  unsigned long long* d;
  cudaMalloc(&d, ctas * 8);
  for (int it = 0; it < 4; ++it) epi_kernel<MODE, DBG, VAR><<<ctas, 320>>>(ep, M, T, d);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(ctas);
  cudaMemcpy(h.data(), d, ctas * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("%-34s T=%d: epilogue %.2f us (median over %d CTAs, max %.2f) err=%s\n", name, T, h[ctas / 2] * 1e-3, ctas,
         h[ctas - 1] * 1e-3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  const int T = 320, H = 5120, hd = 128, nq = 40, nkv = 40, bs = 64;
  const int qkv_rows = (nq + 2 * nkv) * hd;
  // positions: 256 consecutive (a prefill chunk at 768) + 64 decodes at scattered positions
  std::vector<int> pos(T), slot(T);
  for (int t = 0; t < 256; ++t) pos[t] = 768 + t;
  for (int t = 256; t < T; ++t) pos[t] = 1023;
  for (int t = 0; t < T; ++t) slot[t] = t < 256 ? 768 + t : (t - 255) * 1024 + 1023;  // distinct blocks
  int *dpos, *dslot;
  cudaMalloc(&dpos, T * 4);
  cudaMalloc(&dslot, T * 4);
  cudaMemcpy(dpos, pos.data(), T * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dslot, slot.data(), T * 4, cudaMemcpyHostToDevice);
  std::vector<float> th(hd);
  for (int i = 0; i < hd / 2; ++i) {
    const double inv = std::pow(10000.0, -2.0 * i / hd);
    th[2 * i] = static_cast<float>(inv);
    th[2 * i + 1] = static_cast<float>(inv - static_cast<double>(th[2 * i]));
  }
  float* dth;
  cudaMalloc(&dth, hd * 4);
  cudaMemcpy(dth, th.data(), hd * 4, cudaMemcpyHostToDevice);
  const size_t nblocks = 70 * 1024 / bs + 64;
  void *q, *kc, *vc, *f, *h;
  cudaMalloc(&q, static_cast<size_t>(T) * nq * hd * 2);
  cudaMalloc(&kc, nblocks * nkv * bs * hd * 2);
  cudaMalloc(&vc, nblocks * nkv * bs * hd * 2);
  cudaMalloc(&f, static_cast<size_t>(T) * 13824 * 2);
  cudaMalloc(&h, static_cast<size_t>(T) * H * 4);
  cudaMemset(h, 0, static_cast<size_t>(T) * H * 4);
  EpiParams e;
  e.mode = EPI_QKV_ROPE;
  e.out = q;
  e.ldo = nq * hd;
  e.pos = dpos;
  e.slot = dslot;
  e.rope_theta = dth;
  e.kcache = kc;
  e.vcache = vc;
  e.head_dim = hd;
  e.n_q_local = nq;
  e.n_kv_local = nkv;
  e.block_size = bs;
  run<EPI_QKV_ROPE>("QKV + RoPE + KV append (120 tiles)", e, qkv_rows, T, 120);
  run<EPI_QKV_ROPE, false, 1>("  QKV, 2 chunks per TMEM wait", e, qkv_rows, T, 120);
  run<EPI_QKV_ROPE, false, 2>("  QKV, 32-token emitter", e, qkv_rows, T, 120);
  {
    EpiParams d = e;
    d.dbg = 32;
    run<EPI_QKV_ROPE, true>("  QKV, no RoPE math (dbg)", d, qkv_rows, T, 120);
    d.dbg = 8;
    run<EPI_QKV_ROPE, true>("  QKV, no global stores (dbg)", d, qkv_rows, T, 120);
    d.dbg = 0;
    run<EPI_QKV_ROPE, true>("  QKV (dbg instantiation)", d, qkv_rows, T, 120);
    std::vector<int> pd(T), sd(T);
    for (int t = 0; t < T; ++t) { pd[t] = 1000 + 37 * t; sd[t] = (t % 16) * 1024 + 1023; }
    cudaMemcpy(dpos, pd.data(), T * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dslot, sd.data(), T * 4, cudaMemcpyHostToDevice);
    run<EPI_QKV_ROPE>("  QKV, all tokens decode (sincos)", e, qkv_rows, T, 120);
    for (int t = 0; t < T; ++t) { pd[t] = 768 + t; sd[t] = 768 + t; }
    cudaMemcpy(dpos, pd.data(), T * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dslot, sd.data(), T * 4, cudaMemcpyHostToDevice);
    run<EPI_QKV_ROPE>("  QKV, all tokens one prefill chunk", e, qkv_rows, T, 120);
    cudaMemcpy(dpos, pos.data(), T * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dslot, slot.data(), T * 4, cudaMemcpyHostToDevice);
  }
  EpiParams es = e;
  es.mode = EPI_SILU_MUL;
  es.out = f;
  es.ldo = 13824;
  run<EPI_SILU_MUL>("gate||up SiLU*up (148 tiles)", es, 2 * 13824, T, 148);
  run<EPI_SILU_MUL, false, 1>("  SiLU, 2 chunks per TMEM wait", es, 2 * 13824, T, 148);
  EpiParams ea = e;
  ea.mode = EPI_ADD_F32;
  ea.out = h;
  ea.ldo = H;
  run<EPI_ADD_F32>("residual red.add (40 tiles)", ea, H, T, 40);
  run<EPI_ADD_F32, false, 1>("  red.add, 2 chunks per TMEM wait", ea, H, T, 40);
  EpiParams eb = e;
  eb.mode = EPI_STORE_BF16;
  run<EPI_STORE_BF16>("plain bf16 store (120 tiles)", eb, qkv_rows, T, 120);
  return 0;
}

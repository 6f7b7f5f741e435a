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

template <int MODE, bool DBG = false>
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

template <int MODE, bool DBG = false>
void run(const char* name, EpiParams ep, int M, int T, int ctas) {
  unsigned long long* d;
  cudaMalloc(&d, ctas * 8);
  for (int it = 0; it < 4; ++it) epi_kernel<MODE, DBG><<<ctas, 320>>>(ep, M, T, d);
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
  EpiParams ea = e;
  ea.mode = EPI_ADD_F32;
  ea.out = h;
  ea.ldo = H;
  run<EPI_ADD_F32>("residual red.add (40 tiles)", ea, H, T, 40);
  EpiParams eb = e;
  eb.mode = EPI_STORE_BF16;
  run<EPI_STORE_BF16>("plain bf16 store (120 tiles)", eb, qkv_rows, T, 120);
  return 0;
}

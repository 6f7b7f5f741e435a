// Microbenchmark: raw tcgen05.mma issue/execute rate (no memory traffic): kind::f16, bf16 in, fp32
// accumulate, operands in shared memory (garbage), accumulator in TMEM.  1-CTA (M=128) and CTA-pair
// (cta_group::2, M=256) for several N; commits every `per_commit` MMAs to an mbarrier and waits, like
// a GEMM mainloop.  Used to size the GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2308_16369_b200/csrc -o tools/umma_rate tools/umma_rate.cu
#include <cstdio>
#include "common.cuh"

using namespace sarathi;

template <int PAIR, int WARP>
__global__ void __launch_bounds__(128, 1) umma_loop(int N, int iters, int per_commit, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR)
      tmem_alloc_pair(&holder, 512);
    else
      tmem_alloc(&holder, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = 0, t1 = 0;
  if (WARP && warp == 0 && rank == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(PAIR ? 256 : 128, N);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    uint32_t ph = 0;
    t0 = globaltimer_ns();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (PAIR)
          umma_f16_ss_pair_warp(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, 1);
        else
          umma_f16_ss_warp(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, 1);
      }
      if ((i + 4) % per_commit == 0) {
        if (PAIR)
          umma_commit_pair_mc_warp(&bar, 0x1);
        else
          umma_commit_warp(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    t1 = globaltimer_ns();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  if (!WARP && warp == 0 && rank == 0 && lane == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(PAIR ? 256 : 128, N);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    uint32_t ph = 0;
    t0 = globaltimer_ns();
    for (int i = 0; i < iters; ++i) {
      const int k = i & 3;
      if (PAIR)
        umma_f16_ss_pair(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, 1);
      else
        umma_f16_ss(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, 1);
      if ((i + 1) % per_commit == 0) {
        if (PAIR)
          umma_commit_pair_mc(&bar, 0x1);
        else
          umma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    t1 = globaltimer_ns();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

// Pipelined variant (the GEMM mainloop's structure): 8 UMMAs per group (one k-block at N = 2 x 160
// or 4 at N=256), a commit per group onto bars[g % S], and before reusing a stage the issuer waits
// for the commit of the group S earlier — no wait on the group just issued.
__global__ void __launch_bounds__(128, 1) umma_pipe(int N, int per_group, int iters, int S, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t holder;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair(&holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(256, N);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    const unsigned long long t0 = globaltimer_ns();
    int groups = iters / per_group;
    for (int g = 0; g < groups; ++g) {
      const int s = g % S;
      if (g >= S) {
        mbar_wait(&bars[s], ((g / S) - 1) & 1);
        tc_fence_after();
      }
      for (int k = 0; k < per_group; ++k)
        umma_f16_ss_pair_warp(tmem + (k & 1) * 256, make_desc_k_sw128(a + (k & 3) * 32), make_desc_k_sw128(b + (k & 3) * 32),
                              idesc, 1);
      umma_commit_pair_mc_warp(&bars[s], 0x1);
    }
    for (int g = groups - S; g < groups; ++g)
      if (g >= 0) mbar_wait(&bars[g % S], (g / S) & 1);
    const unsigned long long t1 = globaltimer_ns();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// The GEMM's exact issue pattern (k-block = 4 k-steps x {UMMA(d0, A_k, B0_k), UMMA(d0 + off2, A_k,
// B1_k)}, N = 160 each, one commit per k-block onto an S-stage ring), optionally with the other warps
// of the CTA pair spinning on mbarriers the way the GEMM's producer / epilogue warps do.
__global__ void __launch_bounds__(192, 1) umma_gemm_like(int kblocks, int S, int off2, int spin, int rotate, int mask, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint64_t never;
  __shared__ uint32_t holder;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    mbar_init(&never, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(&holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 1 && rank == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(256, 160);
    const unsigned long long t0 = globaltimer_ns();
    for (int g = 0; g < kblocks; ++g) {
      const int s = g % S;
      // rotate: each stage has its own 36 KB operand slot (A 16 KB + B 20 KB), like the GEMM's ring
      const uint32_t a = smem_u32(smem) + (rotate ? s * 36864 : 0), b = a + 16384;
      if (g >= S) {
        mbar_wait(&bars[s], ((g / S) - 1) & 1);
        tc_fence_after();
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        umma_f16_ss_pair_warp(tmem, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, 1);
        umma_f16_ss_pair_warp(tmem + off2, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + 10240 + k * 32), idesc, 1);
      }
      umma_commit_pair_mc_warp(&bars[s], static_cast<uint16_t>(mask));
    }
    for (int g = kblocks - S; g < kblocks; ++g)
      if (g >= 0) mbar_wait(&bars[g % S], (g / S) & 1);
    const unsigned long long t1 = globaltimer_ns();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
    if (spin) {  // release the spinners
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&never), 0));
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&never), 1));
    }
  } else if (spin && warp != 1) {
    if (spin == 1 || lane == 0) mbar_wait(&never, 0);  // spin==1: whole warp polls; 2: lane 0 only
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// Two commits per 8-UMMA group (one per stage of a 2-stage group, as a GEMM with 4 UMMAs per
// k-block would need): is the cost per commit instruction or per commit group?
__global__ void __launch_bounds__(128, 1) umma_two_commits(int N, int iters, int dual, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[16];
  __shared__ uint32_t holder;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair(&holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = holder;
  const int S = 6;  // groups in flight
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(256, N);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    const unsigned long long t0 = globaltimer_ns();
    const int groups = iters / 8;
    for (int g = 0; g < groups; ++g) {
      const int s = g % S;
      if (g >= S) {
        mbar_wait(&bars[2 * s], ((g / S) - 1) & 1);
        if (dual) mbar_wait(&bars[2 * s + 1], ((g / S) - 1) & 1);
        tc_fence_after();
      }
      for (int k = 0; k < 8; ++k) {
        umma_f16_ss_pair_warp(tmem, make_desc_k_sw128(a + (k & 3) * 32), make_desc_k_sw128(b + (k & 3) * 32), idesc, 1);
        if (dual && k == 3) umma_commit_pair_mc_warp(&bars[2 * s + 1], 0x1);  // mid-group commit
      }
      umma_commit_pair_mc_warp(&bars[2 * s], 0x1);
    }
    for (int g = groups - S; g < groups; ++g)
      if (g >= 0) mbar_wait(&bars[2 * (g % S)], (g / S) & 1);
    const unsigned long long t1 = globaltimer_ns();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  const size_t smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(umma_loop<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(umma_loop<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(umma_loop<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(umma_loop<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int warpv = 0; warpv < 2; ++warpv)
  for (int pair = 0; pair < 2; ++pair) {
    for (int N : {64, 128, 160, 256}) {
      for (int per_commit : {4, 8, 64}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(pair ? 2 : 1);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = pair ? 2 : 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e;
        if (warpv)
          e = pair ? cudaLaunchKernelEx(&cfg, umma_loop<1, 1>, N, iters, per_commit, d)
                   : cudaLaunchKernelEx(&cfg, umma_loop<0, 1>, N, iters, per_commit, d);
        else
          e = pair ? cudaLaunchKernelEx(&cfg, umma_loop<1, 0>, N, iters, per_commit, d)
                   : cudaLaunchKernelEx(&cfg, umma_loop<0, 0>, N, iters, per_commit, d);
        cudaDeviceSynchronize();
        unsigned long long ns = 0;
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        const double flops = 2.0 * (pair ? 256 : 128) * N * 16 * iters;
        printf("%s %s N=%3d commit/%2d : %7.1f ns per MMA, %7.1f TFLOP/s per %s (%s)\n", warpv ? "warp-uniform" : "lane0-branch", pair ? "pair M=256" : "cta  M=128",
               N, per_commit, ns / (double)iters, flops / ns / 1e3, pair ? "SM pair" : "SM", cudaGetErrorString(e));
      }
    }
  }
  cudaFuncSetAttribute(umma_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int N : {160, 256})
    for (int pg : {4, 8, 16})
      for (int S : {1, 2, 4, 6}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, umma_pipe, N, pg, iters, S, d);
        cudaDeviceSynchronize();
        unsigned long long ns = 0;
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        const double flops = 2.0 * 256 * N * 16 * iters;
        printf("pipelined pair M=256 N=%3d %2d MMAs/commit, %d stages: %7.1f ns per MMA, %7.1f TFLOP/s per pair (%s)\n", N, pg, S,
               ns / (double)iters, flops / ns / 1e3, cudaGetErrorString(e));
      }
  const size_t smem_big = 5 * 36864 + 1024;
  cudaFuncSetAttribute(umma_gemm_like, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  for (int rotate : {0, 1})
    for (int mask : {1, 3})
    for (int spin : {0, 1}) {
      const int off2 = 160;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2);
      cfg.blockDim = dim3(192);
      cfg.dynamicSmemBytes = smem_big;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int kb = 512;
      cudaError_t e = cudaLaunchKernelEx(&cfg, umma_gemm_like, kb, 5, off2, spin, rotate, mask, d);
      cudaDeviceSynchronize();
      unsigned long long ns = 0;
      cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
      printf("gemm-like pair 2xN=160 rotate=%d mask=%d spin=%d: %7.1f ns per k-block (8 UMMAs) (%s)\n", rotate, mask, spin, ns / (double)kb,
             cudaGetErrorString(e ? e : cudaGetLastError()));
    }
  cudaFuncSetAttribute(umma_two_commits, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int N : {128, 160})
    for (int dual : {0, 1}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, umma_two_commits, N, 4096, dual, d);
      cudaDeviceSynchronize();
      unsigned long long ns = 0;
      cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
      printf("two-commit test pair N=%d dual=%d: %7.1f ns per MMA (%s)\n", N, dual, ns / 4096.0, cudaGetErrorString(e ? e : cudaGetLastError()));
    }
  return 0;
}

// Microbenchmark: the GEMM epilogue's TMEM drain on its own.  One CTA per SM, 320 threads like the
// GEMM (warps 2..9 drain, two warps per TMEM lane quarter, alternate 16-column chunks); each drain
// warp reads `chunks` chunks of 32 lanes x 16 columns with tcgen05.ld.32x32b.{x16,x32,x64} and
// either one load in flight (load; wait; consume) or the next load issued before consuming the
// current one (the GEMM's pipelined drain).  Prints the drain time per CTA (median over CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2308_16369_b200/csrc -o tools/tmem_drain tools/tmem_drain.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include "common.cuh"

using namespace sarathi;

SARATHI_DEVICE void ld_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
      "%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

template <int MODE>  // 0: x16 one in flight, 1: x16 pipelined, 2: x32 one in flight, 3: 0 + bf16
                     // transpose through smem + 16-B global stores (the GEMM's store epilogue), 4: 3 + sincos
__global__ void __launch_bounds__(320, 1) drain(int chunks, unsigned long long* out, float* sink, __nv_bfloat16* gout,
                                                 int ldo) {
  __shared__ uint32_t holder;
  __shared__ __align__(16) uint16_t sbuf_all[8][16 * 32];
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 1) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = globaltimer_ns();
  float acc = 0.f;
  if (warp >= 2) {
    const uint32_t quarter = warp & 3, eh = (warp - 2) >> 2;
    const uint32_t trow = tmem + ((quarter * 32u) << 16);
    if (MODE == 0) {
      for (int ch = eh; ch < chunks; ch += 2) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(trow + (ch % 32) * 16, r);
        tmem_ld_wait_regs(r);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += __uint_as_float(r[j]);
      }
    } else if (MODE == 1) {
      uint32_t r[16];
      tmem_ld_32x32b_x16(trow + eh * 16, r);
      tmem_ld_wait_regs(r);
      for (int ch = eh; ch < chunks; ch += 2) {
        uint32_t n[16];
        const bool more = ch + 2 < chunks;
        if (more) tmem_ld_32x32b_x16(trow + ((ch + 2) % 32) * 16, n);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += __uint_as_float(r[j]);
        if (more) {
          tmem_ld_wait_regs(n);
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = n[j];
        }
      }
    } else if (MODE >= 3) {
      uint16_t* sb = sbuf_all[warp - 2];
      const uint32_t lane = threadIdx.x & 31;
      const int row0 = blockIdx.x * 128 + quarter * 32;
      for (int ch = eh; ch < chunks; ch += 2) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(trow + (ch % 32) * 16, r);
        tmem_ld_wait_regs(r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float x = __uint_as_float(r[j]);
          if (MODE == 4) {
            float sn, cs;
            __sincosf(x * 0.001f + j, &sn, &cs);
            x = x * cs + sn;
          }
          sb[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(x));
        }
        __syncwarp();
        const int g = static_cast<int>(lane & 3), m = row0 + g * 8;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int tok = ch * 16 + pass * 8 + static_cast<int>(lane >> 2);
          *reinterpret_cast<uint4*>(gout + static_cast<size_t>(tok) * ldo + m) =
              *reinterpret_cast<const uint4*>(sb + (pass * 8 + (lane >> 2)) * 32 + g * 8);
        }
        __syncwarp();
      }
    } else {
      for (int ch = 2 * eh; ch < chunks; ch += 4) {
        uint32_t r[32];
        ld_x32(trow + (ch % 32) * 16, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = globaltimer_ns();
  if (threadIdx.x == 64) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(int chunks, int sms) {
  unsigned long long* d;
  float* sink;
  __nv_bfloat16* gout;
  const int ldo = sms * 128;
  cudaMalloc(&d, sms * 8);
  cudaMalloc(&sink, 4096);
  cudaMalloc(&gout, static_cast<size_t>(chunks) * 16 * ldo * 2);
  for (int it = 0; it < 3; ++it) drain<MODE><<<sms, 320>>>(chunks, d, sink, gout, ldo);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), d, sms * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const char* names[] = {"x16, 1 in flight", "x16, pipelined", "x32, 1 in flight", "x16 + smem transpose + stores",
                         "x16 + sincos + transpose + stores"};
  printf("mode %d (%s) chunks %d: drain %.2f us (median over %d CTAs, max %.2f)  err=%s\n", MODE, names[MODE], chunks,
         h[sms / 2] * 1e-3, sms, h[sms - 1] * 1e-3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(gout);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int sms = 148;
  for (int chunks : {20, 32}) {
    run<0>(chunks, sms);
    run<1>(chunks, sms);
    run<2>(chunks, sms);
    run<3>(chunks, sms);
    run<4>(chunks, sms);
  }
  return 0;
}

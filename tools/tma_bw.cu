// Microbenchmark: per-SM ingest bandwidth of cp.async.bulk (1D, bulk copy engine) into shared
// memory with an S-deep mbarrier ring and no compute, from HBM (unique data) and from L2 (a small
// re-read buffer).  Used to size the GEMM pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bw tools/tma_bw.cu && /tmp/tma_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void bulk_stream(const uint8_t* __restrict__ src, size_t src_bytes, size_t per_cta, int chunk, int stages,
                            int l2mode, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nchunks = static_cast<int>(per_cta / chunk);
  const uint8_t* ptr = src + (l2mode ? (static_cast<size_t>(blockIdx.x % 64) * chunk) : static_cast<size_t>(blockIdx.x) * per_cta);
  const uint8_t* wrap = src + src_bytes;
  unsigned long long acc = 0;
  int s = 0;
  uint32_t ph = 0;
  for (int i = 0; i < nchunks + stages; ++i) {
    if (i >= stages) {  // consume chunk i - stages
      uint32_t done = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}\n"
                     : "=r"(done) : "r"(smem_u32(&bars[s])), "r"(ph ^ 1) : "memory");
      } while (!done);
      acc += smem[static_cast<size_t>(s) * chunk];
    }
    if (i < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bars[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       smem_u32(smem + static_cast<size_t>(s) * chunk)),
                   "l"(ptr), "r"(chunk), "r"(smem_u32(&bars[s]))
                   : "memory");
      ptr += chunk;
      if (l2mode && ptr + chunk > wrap) ptr = src;
    }
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  sink[blockIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = static_cast<size_t>(4) << 30;  // 4 GB unique
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int l2mode = 0; l2mode < 2; ++l2mode) {
    for (int chunk : {16384, 32768}) {
      for (int stages : {4, 6}) {
        if (static_cast<size_t>(chunk) * stages > 200 * 1024) continue;
        for (int ctas_per_sm : {1, 2, -2, -4}) {
          if (ctas_per_sm == 2 && static_cast<size_t>(chunk) * stages > 100 * 1024) continue;
          const int grid = ctas_per_sm > 0 ? sms * ctas_per_sm : sms / (-ctas_per_sm);
          const size_t per_cta = (l2mode ? (static_cast<size_t>(64) << 20) : total) / grid / chunk * chunk;
          const size_t l2bytes = static_cast<size_t>(32) << 20;
          const size_t smem = static_cast<size_t>(chunk) * stages + stages * 8 + 64;
          bulk_stream<<<grid, 32, smem>>>(buf, l2bytes, per_cta, chunk, stages, l2mode, sink);
          cudaEventRecord(e0);
          bulk_stream<<<grid, 32, smem>>>(buf, l2bytes, per_cta, chunk, stages, l2mode, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = static_cast<double>(per_cta) * grid;
          const int used = ctas_per_sm > 0 ? sms : grid;
          printf("%s chunk=%6d stages=%2d grid=%4d : %8.1f GB/s total, %6.1f GB/s per active SM (%.1f us)\n",
                 l2mode ? "L2 " : "HBM", chunk, stages, grid, bytes / ms / 1e6, bytes / ms / 1e6 / used, ms * 1e3);
        }
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}

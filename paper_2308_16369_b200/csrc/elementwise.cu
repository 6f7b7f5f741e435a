// The "others" ops of the decoder block (§2.1: "layer normalization, activation
// functions, residual connections") that are not fused into a GEMM epilogue, plus the device
// weight generator.  All memory-bound; vectorised 16-byte accesses, one CTA per token row.
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>

namespace sarathi {

bool carveout_enabled() {
  static const bool on = [] {
    const char* e = getenv("SARATHI_CARVEOUT");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SARATHI_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {

__global__ void embedding_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ E,
                                 float* __restrict__ h, int H) {
  griddep_launch_dependents();
  griddep_wait();  // h is read by the previous step's kernels
  const int t = blockIdx.x;
  const __nv_bfloat16* src = E + static_cast<size_t>(tok[t]) * H;
  float* dst = h + static_cast<size_t>(t) * H;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const uint4 raw = *reinterpret_cast<const uint4*>(src + i);
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
    float4 o0, o1;
    float2 f;
    f = unpack_bf16x2(w[0]); o0.x = f.x; o0.y = f.y;
    f = unpack_bf16x2(w[1]); o0.z = f.x; o0.w = f.y;
    f = unpack_bf16x2(w[2]); o1.x = f.x; o1.y = f.y;
    f = unpack_bf16x2(w[3]); o1.z = f.x; o1.w = f.y;
    *reinterpret_cast<float4*>(dst + i) = o0;
    *reinterpret_cast<float4*>(dst + i + 4) = o1;
  }
}

template <int kThreads>
__device__ float block_sum(float v, float* sred) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) t += sred[w];
  __syncthreads();
  return t;
}

// Wait until every rank's partial of this all-reduce is published (ready[r] >= epoch).
__device__ __forceinline__ void peer_wait(const PeerSum& ps) {
  if (!ps.ready) return;
  if (threadIdx.x == 0) {
    for (int r = 0; r < ps.world; ++r) {
      unsigned int v;
      while (true) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ps.ready + r) : "memory");
        if (static_cast<int>(v - ps.epoch) >= 0) break;
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
}

// sum over ranks (rank order, fp32) of 4 consecutive bf16 partial values at element offset i
__device__ __forceinline__ float4 peer_sum4(const PeerSum& ps, size_t i) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ps.mm) {  // NVLS: the switch returns the rank sum (fp32 accumulate, bf16 result)
    uint32_t r0, r1;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v2.bf16x2 {%0, %1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "l"(ps.mm + i)
                 : "memory");
    const float2 a0 = unpack_bf16x2(r0), a1 = unpack_bf16x2(r1);
    return make_float4(a0.x, a0.y, a1.x, a1.y);
  }
  for (int r = 0; r < ps.world; ++r) {
    const uint2 raw = *reinterpret_cast<const uint2*>(ps.p[r] + i);
    const float2 a0 = unpack_bf16x2(raw.x), a1 = unpack_bf16x2(raw.y);
    a.x += a0.x;
    a.y += a0.y;
    a.z += a1.x;
    a.w += a1.y;
  }
  return a;
}

// RMSNorm(x; g) = x / sqrt(mean(x^2) + eps) * g  (reading O-8), fp32 math, bf16 out.
template <int kThreads, int kVec>
__global__ void __launch_bounds__(kThreads) rmsnorm_kernel(float* __restrict__ h, const PeerSum add,
                                                           const __nv_bfloat16* __restrict__ g,
                                                           __nv_bfloat16* __restrict__ out, const int* __restrict__ rows,
                                                           int H, float eps, unsigned long long* span_start,
                                                           unsigned long long* span_end, const NormFlags fl) {
  __shared__ float sred[kThreads / 32];
  griddep_launch_dependents();
  // g is a weight: fetched before the grid dependency resolves (overlaps the predecessor's tail)
  uint2 gv[kVec];
#pragma unroll
  for (int c = 0; c < kVec; ++c) {
    const int i = (c * kThreads + threadIdx.x) * 4;
    if (i < H) gv[c] = *reinterpret_cast<const uint2*>(g + i);
  }
  if (fl.wait_ctr) {  // flag chaining: the producing GEMM's CTAs finished their residual adds
    if (threadIdx.x == 0) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl.wait_ctr) : "memory");
      const unsigned long long t0 = globaltimer_ns();
      while (static_cast<int>(v - fl.wait_target) < 0) {
        __nanosleep(32);
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl.wait_ctr) : "memory");
        if (globaltimer_ns() - t0 > 4000000000ull) __trap();
      }
    }
    __syncthreads();
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  } else {
    griddep_wait();  // h / add come from the preceding GEMM (PDL)
  }
  peer_wait(add);  // fused all-reduce: every rank's partial published
  if (span_start && threadIdx.x == 0) atomicMin(span_start, globaltimer_ns());
  const int r = blockIdx.x;
  const int row = rows ? rows[r] : r;
  float* x = h + static_cast<size_t>(row) * H;
  // each thread holds kVec chunks of 4 floats in registers (H <= kThreads * 4 * kVec)
  float4 v[kVec];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < kVec; ++c) {
    const int i = (c * kThreads + threadIdx.x) * 4;
    if (i < H) {
      v[c] = *reinterpret_cast<const float4*>(x + i);
      if (add.world) {
        const float4 a = peer_sum4(add, static_cast<size_t>(row) * H + i);
        v[c].x += a.x; v[c].y += a.y; v[c].z += a.z; v[c].w += a.w;
        *reinterpret_cast<float4*>(x + i) = v[c];
      }
      ss += v[c].x * v[c].x + v[c].y * v[c].y + v[c].z * v[c].z + v[c].w * v[c].w;
    }
  }
  const float tot = block_sum<kThreads>(ss, sred);
  const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
  __nv_bfloat16* o = out + static_cast<size_t>(r) * H;
#pragma unroll
  for (int c = 0; c < kVec; ++c) {
    const int i = (c * kThreads + threadIdx.x) * 4;
    if (i < H) {
      const float2 g0 = unpack_bf16x2(gv[c].x), g1 = unpack_bf16x2(gv[c].y);
      uint2 pk;
      pk.x = pack_bf16x2(v[c].x * inv * g0.x, v[c].y * inv * g0.y);
      pk.y = pack_bf16x2(v[c].z * inv * g1.x, v[c].w * inv * g1.y);
      *reinterpret_cast<uint2*>(o + i) = pk;
    }
  }
  if (fl.done_ctr) {  // count this CTA in after its stores (the consumer GEMM's producer waits on it)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(fl.done_ctr, 1u);
  }
  if (span_end && threadIdx.x == 0) atomicMax(span_end, globaltimer_ns());
}

__global__ void residual_add_kernel(float* __restrict__ h, const PeerSum add, size_t n) {
  peer_wait(add);
  for (size_t i = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) * 4; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x * 4) {
    float4 v = *reinterpret_cast<float4*>(h + i);
    const float4 a = peer_sum4(add, i);
    v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
    *reinterpret_cast<float4*>(h + i) = v;
  }
}

__global__ void vocab_permute_kernel(const float* __restrict__ gathered, float* __restrict__ logits, int world,
                                     int R, int Vl, int V) {
  const int r = blockIdx.x;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const int rank = v / Vl, c = v % Vl;
    logits[static_cast<size_t>(r) * V + v] =
        rank < world ? gathered[(static_cast<size_t>(rank) * R + r) * Vl + c] : 0.f;
  }
}

// ---- counter-based generator (spec: synth/__init__.py header; independent implementation) ----
__device__ __forceinline__ unsigned long long splitmix64_dev(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float odd_v(unsigned long long seed, unsigned long long tau, unsigned long long k) {
  const unsigned long long u = splitmix64_dev(seed ^ ((tau << 40) | k)) >> 40;
  const long long v = 2ll * static_cast<long long>(u) - ((1ll << 24) - 1);
  return static_cast<float>(v);  // |v| < 2^24: exact
}

// Tile-major, pre-swizzled GEMM weight layout: the [128 x 64] tile (m-tile, k-block) is 16 KB
// contiguous, tiles ordered (m-tile, k-block) = the order a stream-K CTA consumes them, and inside
// a tile row r's 16-byte chunk j sits at chunk j ^ (r % 8) — the UMMA K-major SWIZZLE_128B image,
// so one 1D bulk copy lands a tile in shared memory ready for tcgen05.mma.
__device__ __forceinline__ size_t packed_index(int r, int c, int cols) {
  const int rr = r & 127, j = (c & 63) >> 3;
  return ((static_cast<size_t>(r >> 7) * (cols >> 6) + (c >> 6)) << 13) + (rr << 6) + ((j ^ (rr & 7)) << 3) + (c & 7);
}

__global__ void weightgen_kernel(__nv_bfloat16* __restrict__ dst, int rows, int cols, const int* __restrict__ tau,
                                 const float* __restrict__ scale, const long long* __restrict__ base,
                                 unsigned long long seed, int packed) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols);
    const int c = static_cast<int>(i % cols);
    const float v = odd_v(seed, static_cast<unsigned long long>(tau[r]),
                          static_cast<unsigned long long>(base[r] + c));
    dst[packed ? packed_index(r, c, cols) : i] = __float2bfloat16_rn(__fmul_rn(v, scale[r]));
  }
}

__global__ void pack_weight_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, int rows,
                                   int cols) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    dst[packed_index(r, c, cols)] = src[i];
  }
}

__global__ void gaingen_kernel(__nv_bfloat16* __restrict__ dst, int n, int tau, long long base,
                               unsigned long long seed, float gscale) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float v = odd_v(seed, static_cast<unsigned long long>(tau), static_cast<unsigned long long>(base + i));
    dst[i] = __float2bfloat16_rn(__fadd_rn(1.0f, __fmul_rn(v, gscale)));
  }
}

}  // namespace

cudaError_t launch_embedding(const int* tok, const __nv_bfloat16* E, float* h, int T, int H, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  launch_pdl(embedding_kernel, dim3(T), dim3(256), 0, st, tok, E, h, H);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm(float* h, const PeerSum& add, const __nv_bfloat16* g, __nv_bfloat16* out,
                           const int* rows, int R, int H, float eps, cudaStream_t st, unsigned long long* span_start,
                           unsigned long long* span_end, const NormFlags& fl) {
  if (R == 0) return cudaSuccess;
  if (H % 4) return cudaErrorInvalidValue;
  // one CTA per row, sized so that every row of a batch (T <= 512) is resident in ONE wave
  // (a second partial wave doubles the latency of this latency-bound kernel)
  if (H <= 256 * 4 * 2) {
    launch_pdl(rmsnorm_kernel<256, 2>, dim3(R), dim3(256), 0, st, h, add, g, out, rows, H, eps, span_start, span_end, fl);
  } else if (H <= 256 * 4 * 5) {
    launch_pdl(rmsnorm_kernel<256, 5>, dim3(R), dim3(256), 0, st, h, add, g, out, rows, H, eps, span_start, span_end, fl);
  } else if (H <= 512 * 4 * 8) {
    launch_pdl(rmsnorm_kernel<512, 8>, dim3(R), dim3(512), 0, st, h, add, g, out, rows, H, eps, span_start, span_end, fl);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_residual_add(float* h, const PeerSum& add, int T, int H, cudaStream_t st) {
  const size_t n = static_cast<size_t>(T) * H;
  if (n == 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<size_t>(1184, (n / 4 + 255) / 256));
  static bool carved = false;
  if (!carved) {
    prefer_max_smem(residual_add_kernel);
    carved = true;
  }
  residual_add_kernel<<<blocks, 256, 0, st>>>(h, add, n);
  return cudaGetLastError();
}

cudaError_t launch_vocab_permute(const float* gathered, float* logits, int world, int R, int Vl, int V,
                                 cudaStream_t st) {
  if (R == 0) return cudaSuccess;
  vocab_permute_kernel<<<R, 256, 0, st>>>(gathered, logits, world, R, Vl, V);
  return cudaGetLastError();
}

cudaError_t launch_weightgen(__nv_bfloat16* dst, int rows, int cols, const int* tau, const float* scale,
                             const long long* base, unsigned long long seed, int packed, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  if (packed && cols % 64) return cudaErrorInvalidValue;
  weightgen_kernel<<<148 * 16, 256, 0, st>>>(dst, rows, cols, tau, scale, base, seed, packed);
  return cudaGetLastError();
}

cudaError_t launch_pack_weight(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int cols, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  if (cols % 64) return cudaErrorInvalidValue;
  pack_weight_kernel<<<148 * 16, 256, 0, st>>>(src, dst, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_gaingen(__nv_bfloat16* dst, int n, int tau, long long base, unsigned long long seed,
                           cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const float gscale = static_cast<float>(0.1 / static_cast<double>(1 << 24));
  gaingen_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, n, tau, base, seed, gscale);
  return cudaGetLastError();
}

}  // namespace sarathi

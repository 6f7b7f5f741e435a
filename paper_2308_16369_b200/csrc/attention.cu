// Attention split by token kind (§4.3: "letting the attention computations for
// the prefill and decodes happen separately. The attention operation for decode requests is
// batched together, while the attention in prefill chunk is processed separately").
//
//  * decode_attention: one query per decode request against its paged KV (keys [0, ctx-1]),
//    split-K over the sequence; each CTA owns (request, kv head, split) and streams whole
//    contiguous KV blocks ([bs x hd] bf16, 16 KB at bs=64, hd=128) into a shared-memory ring with
//    cp.async.bulk + mbarrier (TMA bulk engine), computes q.k with 16-lane dot products and
//    warp-shuffle reductions, and runs the online softmax in fp32 (exp2 domain).  All G = n_q/n_kv
//    query heads of a GQA group share one KV stream.  Partial (o, lse) per split are merged by
//    decode_combine.  HBM-bound by design (decode attention "does not benefit
//    from batch size").
//  * prefill_attention: the chunk's p queries at positions s..s+p-1 against keys [0, s+i]
//    (progressive causal mask, PAPER.md L362-369 Fig. fig-attn-chunk-prefills; inclusive,
//    reading O-9) over the request's paged cache (prefix + the chunk itself, appended by the
//    QKV epilogue).  Flash-style online softmax with mma.sync m16n8k16 bf16 (first version).
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>

namespace sarathi {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// Decode attention
// ---------------------------------------------------------------------------
template <int HD, int G>
__global__ void __launch_bounds__(128)
    decode_attn_kernel(DecodeAttnArgs a) {
  constexpr int kThreads = 128;
  constexpr int kLanesPerKey = HD / 8;            // 16 lanes x 8 dims (HD=128); 8 lanes (HD=64)
  constexpr int kKeyGroups = kThreads / kLanesPerKey;
  const int j = blockIdx.x;           // decode request index
  const int kvh = blockIdx.y;         // kv head (local)
  const int z = blockIdx.z;           // split
  const int bs = a.block_size;
  const int ctx = a.ctx[j];
  const int nblk = (ctx + bs - 1) / bs;
  const int b0 = z * a.blocks_per_split;
  const int b1 = min(nblk, b0 + a.blocks_per_split);
  const int nq = a.n_q_local;
  const int q_head0 = kvh * G;
  const size_t block_bytes = static_cast<size_t>(bs) * HD * 2;

  extern __shared__ __align__(128) uint8_t smem[];
  const int S = a.stages;
  uint8_t* ring = smem;                                                // S x (K block, V block)
  float* s_p = reinterpret_cast<float*>(smem + S * 2 * block_bytes);   // [G][bs]
  float* s_stat = s_p + G * bs;                                        // [G][2] m, scale | [G] sum
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(s_stat + 4 * G) + 7) & ~uintptr_t(7));  // full[S]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int grp = tid / kLanesPerKey, gl = tid % kLanesPerKey;

  float* part_o = a.part_o;   // [d][nq][splits][HD]
  float* part_lse = a.part_lse;  // [d][nq][splits]

  if (b0 >= b1) {
    if (a.splits > 1 && tid < G) {
      part_lse[(static_cast<size_t>(j) * nq + q_head0 + tid) * a.splits + z] = -INFINITY;
    }
    return;
  }

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int* table = a.block_tables + static_cast<size_t>(j) * a.max_blocks;
  const uint8_t* kbase = static_cast<const uint8_t*>(a.kcache);
  const uint8_t* vbase = static_cast<const uint8_t*>(a.vcache);
  const int n_local = b1 - b0;
  uint64_t pol = 0;
  if (tid == 0) {
    pol = policy_evict_first();
    for (int i = 0; i < min(S, n_local); ++i) {
      const size_t blk = static_cast<size_t>(table[b0 + i]) * a.n_kv_local + kvh;
      mbar_arrive_expect_tx(&bars[i], 2 * block_bytes);
      bulk_load_1d(ring + (2 * i) * block_bytes, kbase + blk * block_bytes, block_bytes, &bars[i], pol);
      bulk_load_1d(ring + (2 * i + 1) * block_bytes, vbase + blk * block_bytes, block_bytes, &bars[i], pol);
    }
  }

  // q for all G heads, this lane's 8 dims, pre-scaled by softmax scale * log2(e)
  const float qscale = a.scale * kLog2e;
  float q[G][8];
  {
    const __nv_bfloat16* qrow = a.q + static_cast<size_t>(a.q_row0 + j) * a.q_ld;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint4 raw = *reinterpret_cast<const uint4*>(qrow + (q_head0 + g) * HD + gl * 8);
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(w[i]);
        q[g][2 * i] = f.x * qscale;
        q[g][2 * i + 1] = f.y * qscale;
      }
    }
  }

  // PV ownership: thread owns dims (2*dp, 2*dp+1) for keys with key % 2 == kh
  constexpr int kDimPairs = HD / 2;
  const int dp = tid % kDimPairs;
  const int kh = tid / kDimPairs;              // 0 or 1 (HD=128); 0..3 (HD=64)
  constexpr int kKeyStride = kThreads / kDimPairs;
  float acc[G][2];
  float m_run[G], l_run[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    acc[g][0] = acc[g][1] = 0.f;
    m_run[g] = -INFINITY;
    l_run[g] = 0.f;
  }

  for (int i = 0; i < n_local; ++i) {
    const int s = i % S;
    const uint32_t ph = (i / S) & 1;
    mbar_wait(&bars[s], ph);
    const __nv_bfloat16* Kb = reinterpret_cast<const __nv_bfloat16*>(ring + (2 * s) * block_bytes);
    const __nv_bfloat16* Vb = reinterpret_cast<const __nv_bfloat16*>(ring + (2 * s + 1) * block_bytes);
    const int key0 = (b0 + i) * bs;
    const int nkeys = min(bs, ctx - key0);

    // scores (log2 domain)
    for (int k = grp; k < bs; k += kKeyGroups) {
      const uint4 raw = *reinterpret_cast<const uint4*>(Kb + k * HD + gl * 8);
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
      float kf[8];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(w[t]);
        kf[2 * t] = f.x;
        kf[2 * t + 1] = f.y;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float d = 0.f;
#pragma unroll
        for (int t = 0; t < 8; ++t) d = fmaf(q[g][t], kf[t], d);
#pragma unroll
        for (int off = kLanesPerKey / 2; off >= 1; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        if (gl == 0) s_p[g * bs + k] = (k < nkeys) ? d : -INFINITY;
      }
    }
    __syncthreads();
    // softmax statistics: warp w handles heads w, w+4, ...
    for (int g = warp; g < G; g += 4) {
      float mx = -INFINITY;
      for (int k = lane; k < bs; k += 32) mx = fmaxf(mx, s_p[g * bs + k]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_old = (i == 0) ? -INFINITY : s_stat[2 * g];
      const float m_new = (i == 0) ? mx : fmaxf(m_old, mx);
      float sum = 0.f;
      for (int k = lane; k < bs; k += 32) {
        const float pv = exp2f(s_p[g * bs + k] - m_new);
        s_p[g * bs + k] = pv;
        sum += pv;
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      if (lane == 0) {
        s_stat[2 * g] = m_new;
        s_stat[2 * g + 1] = (i == 0) ? 0.f : exp2f(m_old - m_new);
        s_stat[2 * G + g] = sum;
      }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float sc = s_stat[2 * g + 1];
      const float bsum = s_stat[2 * G + g];
      acc[g][0] *= sc;
      acc[g][1] *= sc;
      l_run[g] = l_run[g] * sc + bsum;
      m_run[g] = s_stat[2 * g];
    }
    for (int k = kh; k < nkeys; k += kKeyStride) {
      const float2 v = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(Vb + k * HD + 2 * dp));
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pv = s_p[g * bs + k];
        acc[g][0] = fmaf(pv, v.x, acc[g][0]);
        acc[g][1] = fmaf(pv, v.y, acc[g][1]);
      }
    }
    __syncthreads();  // stage s and s_p free
    if (tid == 0 && i + S < n_local) {
      const size_t blk = static_cast<size_t>(table[b0 + i + S]) * a.n_kv_local + kvh;
      mbar_arrive_expect_tx(&bars[s], 2 * block_bytes);
      bulk_load_1d(ring + (2 * s) * block_bytes, kbase + blk * block_bytes, block_bytes, &bars[s], pol);
      bulk_load_1d(ring + (2 * s + 1) * block_bytes, vbase + blk * block_bytes, block_bytes, &bars[s], pol);
    }
  }

  // reduce the kKeyStride key-interleaved partial accumulators through shared memory
  float* red = reinterpret_cast<float*>(ring);  // ring is free now: [kKeyStride][G][HD]
#pragma unroll
  for (int g = 0; g < G; ++g) {
    red[(kh * G + g) * HD + 2 * dp] = acc[g][0];
    red[(kh * G + g) * HD + 2 * dp + 1] = acc[g][1];
  }
  __syncthreads();
  for (int idx = tid; idx < G * HD; idx += kThreads) {
    const int g = idx / HD, dd = idx % HD;
    float o = 0.f;
#pragma unroll
    for (int t = 0; t < kKeyStride; ++t) o += red[(t * G + g) * HD + dd];
    const float l = l_run[g];  // identical in every thread
    const int qh = q_head0 + g;
    if (a.splits == 1) {
      a.out[static_cast<size_t>(a.q_row0 + j) * a.out_ld + qh * HD + dd] = __float2bfloat16_rn(o / l);
    } else {
      part_o[((static_cast<size_t>(j) * nq + qh) * a.splits + z) * HD + dd] = o / l;
      if (dd == 0) part_lse[(static_cast<size_t>(j) * nq + qh) * a.splits + z] = m_run[g] + log2f(l);
    }
  }
}

__global__ void decode_combine_kernel(DecodeAttnArgs a, int HD) {
  const int j = blockIdx.x, qh = blockIdx.y;
  const int nq = a.n_q_local;
  const float* lse = a.part_lse + (static_cast<size_t>(j) * nq + qh) * a.splits;
  float mx = -INFINITY;
  for (int z = 0; z < a.splits; ++z) mx = fmaxf(mx, lse[z]);
  float den = 0.f;
  for (int z = 0; z < a.splits; ++z) den += (lse[z] == -INFINITY) ? 0.f : exp2f(lse[z] - mx);
  for (int dd = threadIdx.x; dd < HD; dd += blockDim.x) {
    float o = 0.f;
    for (int z = 0; z < a.splits; ++z) {
      if (lse[z] == -INFINITY) continue;
      o += exp2f(lse[z] - mx) * a.part_o[((static_cast<size_t>(j) * nq + qh) * a.splits + z) * HD + dd];
    }
    a.out[static_cast<size_t>(a.q_row0 + j) * a.out_ld + qh * HD + dd] = __float2bfloat16_rn(o / den);
  }
}

// ---------------------------------------------------------------------------
// Chunked-prefill attention (mma.sync m16n8k16 bf16, fp32 accumulate)
// ---------------------------------------------------------------------------
SARATHI_DEVICE void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SARATHI_DEVICE void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SARATHI_DEVICE void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SARATHI_DEVICE void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
SARATHI_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
SARATHI_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// smem tile [rows][HD] bf16 with 16-byte chunks XOR-swizzled by (row % 8)
template <int HD>
SARATHI_DEVICE uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * (HD * 2) + ((chunk ^ (row & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(128)
    prefill_attn_kernel(PrefillAttnArgs a) {
  constexpr int BQ = 64, BK = 64;
  constexpr int kChunks = HD / 8;  // 16-byte chunks per row
  const int qt = blockIdx.x, qh = blockIdx.y;
  const int kvh = qh * a.n_kv_local / a.n_q_local;
  const int q0 = qt * BQ;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = a.start;          // cached prefix length s
  const int p = a.p;
  const int kv_len = s0 + p;
  const int q_hi = min(q0 + BQ, p);  // exclusive
  const int key_end = s0 + q_hi;     // keys needed: [0, key_end)
  const int ntiles = (key_end + BK - 1) / BK;
  const int bs = a.block_size;

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;                         // BQ x HD
  uint8_t* sK = sQ + BQ * HD * 2;             // 2 x BK x HD
  uint8_t* sV = sK + 2 * BK * HD * 2;         // 2 x BK x HD
  const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK), sVa = smem_u32(sV);

  // load Q tile
  for (int c = tid; c < BQ * kChunks; c += 128) {
    const int r = c / kChunks, ch = c % kChunks;
    const int qi = q0 + r;
    const __nv_bfloat16* src = a.q + static_cast<size_t>(a.q_row0 + min(qi, p - 1)) * a.q_ld + qh * HD + ch * 8;
    cp_async16(sQa + swz<HD>(r, ch), src, qi < p);
  }
  auto load_kv = [&](int tile, int buf) {
    for (int c = tid; c < BK * kChunks; c += 128) {
      const int r = c / kChunks, ch = c % kChunks;
      const int key = tile * BK + r;
      const bool valid = key < kv_len;
      const int kk = valid ? key : 0;
      const int blk = a.block_table[kk / bs];
      const size_t row = (static_cast<size_t>(blk) * a.n_kv_local + kvh) * bs + kk % bs;
      const uint32_t off = buf * BK * HD * 2 + swz<HD>(r, ch);
      cp_async16(sKa + off, static_cast<const __nv_bfloat16*>(a.kcache) + row * HD + ch * 8, valid);
      cp_async16(sVa + off, static_cast<const __nv_bfloat16*>(a.vcache) + row * HD + ch * 8, valid);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const float sl2 = a.scale * kLog2e;
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int qr0 = q0 + warp * 16 + gid;        // this thread's two query rows (chunk-local)
  const int qpos0 = s0 + qr0, qpos1 = qpos0 + 8;
  uint32_t qf[HD / 16][4];

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load_kv(t + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int row = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int ch = kk * 2 + (lane >> 4);
        ldmatrix_x4(sQa + swz<HD>(row, ch), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // S = Q K^T : 16 x 64 per warp
    float sacc[BK / 8][4];
#pragma unroll
    for (int n = 0; n < BK / 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
    const uint32_t kb = sKa + buf * BK * HD * 2;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int n2 = 0; n2 < BK / 16; ++n2) {
        const int row = n2 * 16 + (lane & 7) + 8 * (lane >> 4);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(kb + swz<HD>(row, ch), b0, b1, b2, b3);
        mma_bf16_16816(sacc[2 * n2], qf[kk], b0, b1);
        mma_bf16_16816(sacc[2 * n2 + 1], qf[kk], b2, b3);
      }
    }
    // mask + online softmax (log2 domain)
    const int kbase = t * BK;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < BK / 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + 2 * tig + (e & 1);
        const int qp = (e < 2) ? qpos0 : qpos1;
        float v = sacc[n][e] * sl2;
        if (key > qp) v = -INFINITY;
        sacc[n][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
    float scale[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mnew = fmaxf(mrow[r], mx[r]);
      scale[r] = (mnew == -INFINITY) ? 1.f : exp2f(mrow[r] - mnew);
      mrow[r] = mnew;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int n = 0; n < BK / 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = mrow[e >> 1];
        const float pv = (m == -INFINITY) ? 0.f : exp2f(sacc[n][e] - m);
        sacc[n][e] = pv;
        rs[e >> 1] += pv;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      lrow[r] = lrow[r] * scale[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= scale[0];
      o[i][1] *= scale[0];
      o[i][2] *= scale[1];
      o[i][3] *= scale[1];
    }
    // O += P V
    const uint32_t vb = sVa + buf * BK * HD * 2;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16x2(sacc[2 * kk][0], sacc[2 * kk][1]);
      pa[1] = pack_bf16x2(sacc[2 * kk][2], sacc[2 * kk][3]);
      pa[2] = pack_bf16x2(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
      pa[3] = pack_bf16x2(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
      for (int n2 = 0; n2 < HD / 16; ++n2) {
        const int row = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int ch = n2 * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(vb + swz<HD>(row, ch), b0, b1, b2, b3);
        mma_bf16_16816(o[2 * n2], pa, b0, b1);
        mma_bf16_16816(o[2 * n2 + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // write O rows (bf16)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = qr0 + 8 * r;
    if (qi >= p) continue;
    const float inv = 1.f / lrow[r];
    __nv_bfloat16* dst = a.out + static_cast<size_t>(a.q_row0 + qi) * a.out_ld + qh * HD;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      const int col = n * 8 + 2 * tig;
      *reinterpret_cast<uint32_t*>(dst + col) = pack_bf16x2(o[n][2 * r] * inv, o[n][2 * r + 1] * inv);
    }
  }
}

template <int HD, int G>
cudaError_t launch_decode_t(const DecodeAttnArgs& a, cudaStream_t st) {
  const size_t block_bytes = static_cast<size_t>(a.block_size) * HD * 2;
  const size_t smem = a.stages * 2 * block_bytes + (G * a.block_size + 4 * G + 8) * sizeof(float) + 8 * a.stages + 16;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(decode_attn_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  dim3 grid(a.d, a.n_kv_local, a.splits);
  decode_attn_kernel<HD, G><<<grid, 128, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1) return e;
  decode_combine_kernel<<<dim3(a.d, a.n_q_local), 128, 0, st>>>(a, HD);
  return cudaGetLastError();
}

template <int HD>
cudaError_t launch_decode_hd(const DecodeAttnArgs& a, cudaStream_t st) {
  const int G = a.n_q_local / a.n_kv_local;
  switch (G) {
    case 1: return launch_decode_t<HD, 1>(a, st);
    case 2: return launch_decode_t<HD, 2>(a, st);
    case 4: return launch_decode_t<HD, 4>(a, st);
    case 8: return launch_decode_t<HD, 8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

size_t decode_smem_bytes(int head_dim, int block_size, int stages, int G) {
  return stages * 2 * static_cast<size_t>(block_size) * head_dim * 2 + (G * block_size + 4 * G + 8) * sizeof(float) +
         8 * stages + 16;
}

cudaError_t launch_decode_attention(const DecodeAttnArgs& a, cudaStream_t st) {
  if (a.d == 0) return cudaSuccess;
  if (a.head_dim == 128) return launch_decode_hd<128>(a, st);
  if (a.head_dim == 64) return launch_decode_hd<64>(a, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, cudaStream_t st) {
  if (a.p == 0) return cudaSuccess;
  dim3 grid((a.p + 63) / 64, a.n_q_local);
  if (a.head_dim == 128) {
    const size_t smem = (64 + 4 * 64) * 128 * 2;
    static bool c = false;
    if (!c) {
      cudaFuncSetAttribute(prefill_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      c = true;
    }
    prefill_attn_kernel<128><<<grid, 128, smem, st>>>(a);
  } else if (a.head_dim == 64) {
    const size_t smem = (64 + 4 * 64) * 64 * 2;
    prefill_attn_kernel<64><<<grid, 128, smem, st>>>(a);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace sarathi

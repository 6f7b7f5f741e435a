// Attention split by token kind (§4.3: "letting the attention computations for
// the prefill and decodes happen separately. The attention operation for decode requests is
// batched together, while the attention in prefill chunk is processed separately").
//
//  * decode_attn_mma: one query per decode request against its paged KV (keys [0, ctx-1]), split-K
//    over the sequence when there are few requests; each CTA owns (request, kv head, split), a
//    producer warp TMA-loads whole (block, head) K and V tiles (SW128) into a 3-stage ring, and 4
//    compute warps run QK^T / PV with mma.sync (the G query heads of a GQA group are the MMA rows)
//    and a per-warp online softmax merged once.  Partial (o, lse) per split are merged by
//    decode_combine.  HBM-bound by design (decode attention "does not benefit from
//    batch size"); it streams at ~0.97 of the measured HBM copy bandwidth.
//  * prefill_attn_tc: the chunk's p queries at positions s..s+p-1 against keys [0, s+i]
//    (progressive causal mask, PAPER.md L362-369 Fig. fig-attn-chunk-prefills; inclusive, reading
//    O-9) over the request's paged cache (prefix + the chunk itself, appended by the QKV epilogue),
//    on the 5th-gen tensor cores: S and O accumulate in TMEM, P goes through shared memory.
//    Every block size alloc_kv accepts (16/32/64/128) divides its 128-key tile.
#include "common.cuh"
#include "kernels.cuh"
#include "gemm.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace sarathi {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// mma.sync / ldmatrix / cp.async helpers
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
SARATHI_DEVICE float ex2_approx(float x) {  // 2^x, MUFU.EX2 (x = -inf -> 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SARATHI_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
SARATHI_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }


// ---------------------------------------------------------------------------
// Decode attention (paged KV, split-K over the sequence)
//   grid (d, n_kv_local, splits); 160 threads: warps 0-3 compute, warp 4 = TMA producer.
//   Each KV block (bs keys x hd) of K and of V is one 2D TMA load (128B swizzle) into an S-stage
//   ring.  Compute warp w owns the 16-key groups w, w+4, ... of every block and runs, per group,
//   S = Q K^T (mma.sync m16n8k16; the G query heads of the GQA group are the MMA rows, padded to
//   16), its own online softmax (fp32, exp2 domain) and O += P V.  The four warps' (m, l, O) are
//   merged once at the end; splits > 1 write (o, lse) partials for decode_combine.
// ---------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(160)
    decode_attn_mma(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                    DecodeAttnArgs a) {
  griddep_launch_dependents();
  if (!a.wait_at_end) griddep_wait();  // q comes from the QKV GEMM (PDL)
  const bool last_cta = blockIdx.x == gridDim.x - 1 && blockIdx.y == gridDim.y - 1 && blockIdx.z == gridDim.z - 1;
  if (a.span_start && threadIdx.x == 0) atomicMin(a.span_start, globaltimer_ns());
  constexpr int NBOX = HD / 64;  // 128-byte TMA boxes per row
  const int j = blockIdx.x, kvh = blockIdx.y, z = blockIdx.z;
  const int G = a.n_q_local / a.n_kv_local;
  const int bs = a.block_size;
  const int ctx = a.ctx[j];
  const int nblk = (ctx + bs - 1) / bs;
  const int b0 = z * a.blocks_per_split;
  const int b1 = min(nblk, b0 + a.blocks_per_split);
  const int nq = a.n_q_local;
  const int q_head0 = kvh * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;

  if (b0 >= b1) {
    if (a.splits > 1 && tid < G)
      a.part_lse[(static_cast<size_t>(j) * nq + q_head0 + tid) * a.splits + z] = -INFINITY;
    if (a.wait_at_end && last_cta) griddep_wait();
    return;
  }
  const int S = a.stages;
  const uint32_t half_bytes = static_cast<uint32_t>(bs) * 128;       // one 64-col box of a block
  const uint32_t blk_bytes = half_bytes * NBOX;                       // K (or V) block
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * 2 * blk_bytes);
  uint64_t* empty = full + S;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);  // one arrive per compute warp
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int n_local = b1 - b0;
  const int* table = a.block_tables + static_cast<size_t>(j) * a.max_blocks;

  if (warp == 4) {
    // ---------------- producer (warp-uniform; elected lane issues) ----------------
    if (lane == 0) {
      tma_prefetch_desc(&mapK);
      tma_prefetch_desc(&mapV);
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < n_local; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        const int row0 = (table[b0 + i] * a.n_kv_local + kvh) * bs;
        uint8_t* kd = smem + static_cast<size_t>(s) * 2 * blk_bytes;
        uint8_t* vd = kd + blk_bytes;
        mbar_arrive_expect_tx(&full[s], 2 * blk_bytes);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx) {
          tma_load_2d(kd + bx * half_bytes, &mapK, &full[s], bx * 64, row0, pol);
          tma_load_2d(vd + bx * half_bytes, &mapV, &full[s], bx * 64, row0, pol);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- compute warps ----------------
  const float sl2 = a.scale * kLog2e;
  // Q fragment (A operand, 16 x HD): row = head within the group (rows >= G are zero)
  uint32_t qf[HD / 16][4];
  {
    const __nv_bfloat16* qrow = a.q + static_cast<size_t>(a.q_row0 + j) * a.q_ld + static_cast<size_t>(q_head0) * HD;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int c0 = kk * 16 + 2 * tig;
      qf[kk][0] = gid < G ? *reinterpret_cast<const uint32_t*>(qrow + static_cast<size_t>(gid) * HD + c0) : 0u;
      qf[kk][1] = gid + 8 < G ? *reinterpret_cast<const uint32_t*>(qrow + static_cast<size_t>(gid + 8) * HD + c0) : 0u;
      qf[kk][2] = gid < G ? *reinterpret_cast<const uint32_t*>(qrow + static_cast<size_t>(gid) * HD + c0 + 8) : 0u;
      qf[kk][3] = gid + 8 < G ? *reinterpret_cast<const uint32_t*>(qrow + static_cast<size_t>(gid + 8) * HD + c0 + 8) : 0u;
    }
  }
  float o[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int ngroups = bs / 16;
  int s = 0;
  uint32_t ph = 0;
  for (int i = 0; i < n_local; ++i) {
    mbar_wait(&full[s], ph);
    const uint32_t kb = smem_u32(smem + static_cast<size_t>(s) * 2 * blk_bytes);
    const uint32_t vb = kb + blk_bytes;
    const int key_base = (b0 + i) * bs;
    for (int grp = warp; grp < (a.dbg & 1 ? 0 : ngroups); grp += 4) {
      const int k0 = grp * 16;  // key row within the block
      float sacc[2][4];
#pragma unroll
      for (int n = 0; n < 2; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int row = k0 + (lane & 7) + 8 * (lane >> 4);
        const int ch = kk * 2 + ((lane >> 3) & 1);  // 16-B chunk in the row
        const uint32_t addr = kb + (ch >> 3) * half_bytes + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        uint32_t b0r, b1r, b2r, b3r;
        ldmatrix_x4(addr, b0r, b1r, b2r, b3r);
        mma_bf16_16816(sacc[0], qf[kk], b0r, b1r);
        mma_bf16_16816(sacc[1], qf[kk], b2r, b3r);
      }
      // scale to the log2 domain; keys >= ctx masked (only the request's last block has any)
      float mx[2] = {-INFINITY, -INFINITY};
      const bool tail = key_base + bs > ctx;
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = key_base + k0 + n * 8 + 2 * tig + (e & 1);
          const float v = (!tail || key < ctx) ? sacc[n][e] * sl2 : -INFINITY;
          sacc[n][e] = v;
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
      // lazily refreshed running max (FA4 rule): a row keeps a stale m until its max exceeds it by
      // more than 8 (p <= 2^8).  The quad reduction and the O rescale run only when some lane of the
      // warp saw such a max; the row sums stay per-lane partials (reduced once, at the merge).
      float sc[2] = {1.f, 1.f};
      if (__any_sync(0xffffffffu, mx[0] > mrow[0] + 8.f || mx[1] > mrow[1] + 8.f)) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
          if (mx[r] > mrow[r] + 8.f) {  // also the first finite max (mrow = -inf); quad-uniform
            sc[r] = (mrow[r] == -INFINITY) ? 1.f : exp2f(mrow[r] - mx[r]);
            mrow[r] = mx[r];
          }
        }
#pragma unroll
        for (int n = 0; n < HD / 8; ++n) {
          o[n][0] *= sc[0];
          o[n][1] *= sc[0];
          o[n][2] *= sc[1];
          o[n][3] *= sc[1];
        }
      }
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float m = mrow[e >> 1];
          const float pv = (m == -INFINITY) ? 0.f : ex2_approx(sacc[n][e] - m);
          sacc[n][e] = pv;
          lrow[e >> 1] = (e & 1) || n ? lrow[e >> 1] + pv : lrow[e >> 1] * sc[e >> 1] + pv;
        }
      uint32_t pa[4];
      pa[0] = pack_bf16x2(sacc[0][0], sacc[0][1]);
      pa[1] = pack_bf16x2(sacc[0][2], sacc[0][3]);
      pa[2] = pack_bf16x2(sacc[1][0], sacc[1][1]);
      pa[3] = pack_bf16x2(sacc[1][2], sacc[1][3]);
#pragma unroll
      for (int n2 = 0; n2 < HD / 16; ++n2) {
        const int row = k0 + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int ch = n2 * 2 + (lane >> 4);
        const uint32_t addr = vb + (ch >> 3) * half_bytes + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        uint32_t b0r, b1r, b2r, b3r;
        ldmatrix_x4_trans(addr, b0r, b1r, b2r, b3r);
        mma_bf16_16816(o[2 * n2], pa, b0r, b1r);
        mma_bf16_16816(o[2 * n2 + 1], pa, b2r, b3r);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }

  // ---------------- merge the 4 warps' partial softmax states ----------------
#pragma unroll
  for (int r = 0; r < 2; ++r) {  // per-lane partial row sums -> the row's sum over its 4 lanes
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  named_bar_sync(1, 128);  // all compute warps done with the ring
  float* sm_m = reinterpret_cast<float*>(smem);  // [4][16]
  float* sm_l = sm_m + 64;                       // [4][16]
  float* sm_o = sm_l + 64;                       // [4][16][HD]
  if (tig == 0) {
    sm_m[warp * 16 + gid] = mrow[0];
    sm_m[warp * 16 + gid + 8] = mrow[1];
    sm_l[warp * 16 + gid] = lrow[0];
    sm_l[warp * 16 + gid + 8] = lrow[1];
  }
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    const int col = n * 8 + 2 * tig;
    sm_o[(warp * 16 + gid) * HD + col] = o[n][0];
    sm_o[(warp * 16 + gid) * HD + col + 1] = o[n][1];
    sm_o[(warp * 16 + gid + 8) * HD + col] = o[n][2];
    sm_o[(warp * 16 + gid + 8) * HD + col + 1] = o[n][3];
  }
  named_bar_sync(1, 128);
  for (int idx = tid; idx < G * HD; idx += 128) {
    const int g = idx / HD, dd = idx % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w * 16 + g]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = sm_m[w * 16 + g];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      L += sm_l[w * 16 + g] * f;
      O += sm_o[(w * 16 + g) * HD + dd] * f;
    }
    const int qh = q_head0 + g;
    if (a.splits == 1) {
      a.out[static_cast<size_t>(a.q_row0 + j) * a.out_ld + qh * HD + dd] = __float2bfloat16_rn(O / L);
    } else {
      a.part_o[((static_cast<size_t>(j) * nq + qh) * a.splits + z) * HD + dd] = O / L;
      if (dd == 0) a.part_lse[(static_cast<size_t>(j) * nq + qh) * a.splits + z] = M + log2f(L);
    }
  }
  if (a.head_flag) {  // publish this KV head's rows once all d requests' CTAs wrote them
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");  // read by the O GEMM's TMA loads
    named_bar_sync(1, 128);
    if (tid == 0) {
      const int old = atomicAdd(a.head_cnt + kvh, 1);
      if (old == a.d - 1) {
        a.head_cnt[kvh] = 0;  // re-arm for the next launch
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.head_flag + kvh), "r"(a.epoch) : "memory");
      }
    }
  }
  // attention chain: the grid must not complete before the prefill grid; one CTA waiting is
  // enough (the others keep their SM slots free for the rest of the grid)
  if (a.wait_at_end && last_cta) griddep_wait();
  if (a.span_end && threadIdx.x == 0) atomicMax(a.span_end, globaltimer_ns());
}

__global__ void decode_combine_kernel(DecodeAttnArgs a, int HD) {
  griddep_launch_dependents();
  griddep_wait();
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
// Chunked-prefill attention on the 5th-gen tensor cores (tcgen05 / TMEM / TMA).
//   CTA = (128-query tile of the chunk, query head); 256 threads, query row r = TMEM lane r is
//   owned by two threads (one per 64-key / hd/2 column half).  Per key tile t (128 keys = 128/bs paged blocks, TMA-loaded K-major SW128):
//     S_t  = Q K_t^T        UMMA M=128, N=128, K=hd into TMEM (two S buffers: S_{t+1} is issued
//                           before the softmax of S_t, so the tensor core overlaps the softmax)
//     P_t  = exp2(S_t*c - m) bf16 -> smem (K-major SW128, the A operand of the next UMMA)
//     O_t  = P_t V_t        UMMA M=128, N=hd, K=128 keys, B = V tile read MN-major (no transpose)
//     O    = O * alpha + O_t  in registers (online softmax, fp32; reading O-9: key j <= s + i)
//   Issue (TMA + UMMA) is warp 0, warp-uniform with one elected lane.
// ---------------------------------------------------------------------------
constexpr int kPBQ = 128;  // queries per CTA
constexpr int kMaxKsplit = 8;  // key-range split of one (q-tile, head) pair (PrefillAttnArgs::ksplit)

// MN-major SW128 UMMA smem descriptor: 64-element (128 B) rows along MN, MN atoms LBO apart,
// 8-row K groups SBO apart (CuTe canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-B units).
SARATHI_DEVICE uint64_t make_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// BK = keys per tile.  BK = 128 (default): 1 CTA per SM (197 KB smem at HD 128, 512 TMEM columns).
// BK = 64: 256 TMEM columns and <= 100 KB smem (V single-buffered at HD 128), so a prefill CTA leaves
// room on its SM for the decode-attention CTAs running concurrently on the other stream.
template <int HD, int BK, bool PT>
struct PtcSmem {
  static constexpr bool kVdb = BK == 128 || HD == 64;  // V double-buffered
  static constexpr uint32_t kQ = kPBQ * HD * 2;   // Q tile  [HD/64][128 rows][64] SW128
  static constexpr uint32_t kKV = BK * HD * 2;    // K or V tile [HD/64][BK keys][64]
  static constexpr uint32_t kP = PT ? 0 : kPBQ * BK * 2;  // P [BK/64][128 rows][64 keys] (PT: in TMEM)
  static constexpr uint32_t kRed = 2 * kPBQ * 4;  // per-half row maxima / sums
  static constexpr uint32_t kTotal = kQ + (kVdb ? 4 : 3) * kKV + kP + kRed + 256 + 1024;  // + barriers + align slack
  static constexpr uint32_t kTmemCols = BK == 128 ? 512 : 256;
};


// 256 threads: warp w owns TMEM lane quarter (w & 3) -> query rows 32(w&3)..+31, and column half
// ch = w >> 2 of every S tile (keys 64ch..64ch+63) and of O (dims (hd/2)ch..); the two halves of a
// row exchange their maxima through shared memory once per tile.
//
// PT (P in TMEM, BK = 128): three S buffers + O fill the 512 columns; P_t is written bf16-packed
// over the columns of S_t the same thread just read and feeds PV_t as the TMEM A operand, so the
// softmax of tile t never waits for PV_{t-1} (only an O rescale does), and there is no P smem
// image, proxy fence or smem traffic.  S_{t+1} goes to buffer (t+1) mod 3, whose P_{t-2} was
// consumed by PV_{t-2}, which warp 0 waited for before the tile-(t-1) barrier.
template <int HD, int BK, bool PT>
__global__ void __launch_bounds__(256, BK == 128 ? 1 : 2)
    prefill_attn_tc(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                    const __grid_constant__ CUtensorMap mapV, const PrefillAttnArgs a) {
  static_assert(!PT || BK == 128, "P in TMEM needs the 128-key tile");
  using L = PtcSmem<HD, BK, PT>;
  constexpr int kHalves = HD / 64;
  constexpr int kOC = HD / 2;  // O columns per column half
  constexpr int kCH = BK / 2;  // S columns (keys) per column half
  constexpr int kNC = kCH / 16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + L::kQ;          // [2 buffers]
  uint8_t* sV = sK + 2 * L::kKV;     // [2 buffers] (kVdb) or [1]
  uint8_t* sP = sV + (L::kVdb ? 2 : 1) * L::kKV;
  float* red = reinterpret_cast<float*>(sP + L::kP);  // [2 halves][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(red) + L::kRed);
  uint64_t* q_full = bars;        // 1
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* v_full = bars + 3;    // [2]
  uint64_t* s_done = bars + 5;    // [2] ([3] with PT)
  uint64_t* o_done = bars + 8;    // 1
  uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 9);

  const uint32_t warp = warp_id_uniform(), lane = lane_id();
  const uint32_t quarter = warp & 3, chh = warp >> 2;
  const int r = static_cast<int>(quarter * 32 + lane);  // query row within the tile == TMEM lane
  const int s0 = a.start, p = a.p, bs = a.block_size;
  const int kv_len = s0 + p;
  const int last_blk = (kv_len - 1) / bs;      // last block of the request holding valid keys
  const int ntq = (p + kPBQ - 1) / kPBQ;
  const int ksplit = a.ksplit > 1 ? a.ksplit : 1;
  const int n_items = ntq * a.n_q_local * ksplit;
  int& s_merge = *reinterpret_cast<int*>(bars + 10);  // key split: "this CTA merges the pair"
  const bool tr0 = a.trace && blockIdx.x == 0 && threadIdx.x == 0;

  // PDL (attention chain): wait for the QKV GEMM, THEN let the decode attention launch, so the
  // decode grid starts only after q / K / V are complete
  griddep_wait();
  griddep_launch_dependents();
  if (tr0) a.trace[254] = globaltimer_ns();
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 384) a.trace[256 + 2 * blockIdx.x] = globaltimer_ns();
  if (a.span_start && threadIdx.x == 0) atomicMin(a.span_start, globaltimer_ns());
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(holder, L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  auto tS = [&](int b) { return tmem + static_cast<uint32_t>(b * BK); };  // S buffer b
  const uint32_t tO = tmem + (PT ? 3 : 2) * BK;
  auto sbuf = [](int g) { return PT ? g % 3 : g & 1; };          // S buffer of key tile g
  auto sphase = [](int g) { return PT ? (g / 3) & 1 : (g >> 1) & 1; };
  // the CTA walks (q-tile, head) items it = blockIdx.x, + gridDim.x, ...; g = the CTA's running
  // key-tile count, so every ring barrier keeps one phase sequence across items
  int g0 = 0, n_done = 0;
  for (int it = static_cast<int>(blockIdx.x); it < n_items; it += static_cast<int>(gridDim.x), ++n_done) {
  const int qt = it % ntq, qh = (it / ntq) % a.n_q_local, ks = it / (ntq * a.n_q_local);
  const int kvh = qh * a.n_kv_local / a.n_q_local;
  const int q0 = qt * kPBQ;
  const int key_end = s0 + min(q0 + kPBQ, p);  // keys this tile needs: [0, key_end)
  const int ntiles_all = (key_end + BK - 1) / BK;
  const int tb0 = ks * ntiles_all / ksplit;  // this item's key tiles [tb0, tb0 + ntiles)
  const int ntiles = (ks + 1) * ntiles_all / ksplit - tb0;

  // K (or V) tile load: every paged block of the tile (indices past the request clamp to its last
  // block, so every smem byte the UMMAs read is finite; those keys are masked).  K_t is free once
  // S_t is done, V_t once PV_t is done, so they are refilled at different points.
  auto load_tile = [&](int t, int buf, bool is_v) {
    uint64_t* bar = is_v ? &v_full[buf] : &k_full[buf];
    uint8_t* dst = (is_v ? sV : sK) + buf * L::kKV;
    const CUtensorMap* map = is_v ? &mapV : &mapK;
    mbar_arrive_expect_tx_warp(bar, BK * HD * 2);
    for (int kb = 0; kb < BK; kb += bs) {
      const int bi = min(((tb0 + t) * BK + kb) / bs, last_blk);
      const int row = (a.block_table[bi] * a.n_kv_local + kvh) * bs;
#pragma unroll
      for (int h = 0; h < kHalves; ++h) tma_load_2d_warp(dst + h * (BK * 128) + kb * 128, map, bar, h * 64, row);
    }
  };
  const uint32_t idesc_s = make_idesc_bf16_f32(kPBQ, BK);
  const uint32_t idesc_o = make_idesc_bf16_f32(kPBQ, HD) | (1u << 16);  // B (V) MN-major
  auto issue_s = [&](int t) {  // S_t = Q K_t^T into tS[sbuf(g0 + t)]
    const int g = g0 + t, buf = g & 1, sb = sbuf(g);
    mbar_wait(&k_full[buf], (g >> 1) & 1);
    tc_fence_after();
    const uint32_t qa = smem_u32(sQ), kb = smem_u32(sK + buf * L::kKV);
    if (HD == 128 && a.mma8) {  // the 8 k16 steps in one asm block (one elect; GEMM finding)
      umma8_ss_halves(tS(sb), make_desc_k_sw128(qa), (kPBQ * 128) >> 4, make_desc_k_sw128(kb), (BK * 128) >> 4, idesc_s, 0u);
    } else {
#pragma unroll
      for (int k = 0; k < HD / 16; ++k) {
        const uint32_t off = (k >> 2) * (kPBQ * 128) + (k & 3) * 32;  // hd half, 32 B step in the row
        umma_f16_ss_warp(tS(sb), make_desc_k_sw128(qa + off), make_desc_k_sw128(kb + (k >> 2) * (BK * 128) + (k & 3) * 32),
                         idesc_s, k > 0 ? 1u : 0u);
      }
    }
    umma_commit_warp(&s_done[sb]);
  };

  if (warp == 0) {
    mbar_arrive_expect_tx_warp(q_full, L::kQ);
#pragma unroll
    for (int h = 0; h < kHalves; ++h)
      tma_load_2d_warp(sQ + h * (kPBQ * 128), &mapQ, q_full, qh * HD + h * 64, a.q_row0 + q0);
    load_tile(0, g0 & 1, false);
    load_tile(0, L::kVdb ? (g0 & 1) : 0, true);
    if (ntiles > 1) {
      load_tile(1, (g0 + 1) & 1, false);
      if (L::kVdb) load_tile(1, (g0 + 1) & 1, true);
    }
    mbar_wait(q_full, n_done & 1);
    issue_s(0);
  }

  const float c2 = a.scale * kLog2e;
  const int qpos = s0 + q0 + r;  // absolute position of this row's query
  // online softmax with a lazily refreshed running max (the FA4 rule): P = exp2(S c2 - m) is used
  // with a stale m until the tile max exceeds it by more than 8 (P <= 2^8, exact in fp32/bf16
  // range); O accumulates in TMEM across tiles and is rescaled there only when m moves
  float m = -INFINITY, l = 0.f;  // l: this column half's partial row sum
  const uint32_t lane_off = (quarter * 32u) << 16;
  // this row's slice of P: k-block chh (BK 128) or 16-B chunks 4chh.. of the one k-block (BK 64)
  uint8_t* prow = sP + (BK == 128 ? chh * (kPBQ * 128) : 0) + r * 128;
  const int chunk0 = BK == 128 ? 0 : 4 * static_cast<int>(chh);
  const int c_key0 = static_cast<int>(chh) * kCH;

  for (int t = 0; t < ntiles; ++t) {
    const int g = g0 + t, buf = g & 1, sb = sbuf(g);
    const bool tr = tr0 && n_done == 0 && t < 32;
    if (tr) a.trace[t * 8 + 0] = globaltimer_ns();
    if (warp == 0 && t + 1 < ntiles) issue_s(t + 1);  // overlaps this tile's softmax
    mbar_wait(&s_done[sb], sphase(g));
    tc_fence_after();
    if (tr) a.trace[t * 8 + 1] = globaltimer_ns();
    if (warp == 0 && t + 2 < ntiles) load_tile(t + 2, buf, false);  // K_t consumed by S_t
    // this half of the S row in registers: 4 loads in flight, one wait
    uint32_t sr[kNC][16];
#pragma unroll
    for (int c = 0; c < kNC; ++c) tmem_ld_32x32b_x16(tS(sb) + lane_off + c_key0 + c * 16, sr[c]);
#pragma unroll
    for (int c = 0; c < kNC; ++c) tmem_ld_wait_regs(sr[c]);
    const int kbase = (tb0 + t) * BK + c_key0;
    const bool need_mask = (tb0 + t) * BK + BK - 1 > s0 + q0;  // (CTA-uniform) some key lies past a query
    float mt = -INFINITY;
    if (need_mask) {
#pragma unroll
      for (int c = 0; c < kNC; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float v = __uint_as_float(sr[c][j]);
          mt = kbase + c * 16 + j <= qpos ? fmaxf(mt, v) : mt;
        }
    } else {
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < kNC; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(sr[c][j]));
      mt = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    }
    red[chh * kPBQ + r] = mt;
    // PV_{t-1} must be complete before P is overwritten and before O is rescaled
    if (!PT && t > 0) {
      mbar_wait(o_done, (g - 1) & 1);
      tc_fence_after();
      if (warp == 0) {  // V_{t-1} consumed by PV_{t-1}
        if (L::kVdb) {
          if (t + 1 < ntiles) load_tile(t + 1, (g + 1) & 1, true);
        } else {
          load_tile(t, 0, true);
        }
      }
    }
    named_bar_sync(1, 256);  // both halves' maxima posted
    mt = fmaxf(mt, red[(chh ^ 1) * kPBQ + r]) * c2;
    if (tr) a.trace[t * 8 + 2] = globaltimer_ns();
    const bool refresh = mt > m + 8.f;  // also true on the first tile (m = -inf)
    if (t > 0 && __any_sync(0xffffffffu, refresh)) {  // warp-collective TMEM rescale of this O half
      if (PT) {  // PV_{t-1} must be complete
        mbar_wait(o_done, (g - 1) & 1);
        tc_fence_after();
      }
      const float alpha = refresh ? ex2_approx(m - mt) : 1.f;
#pragma unroll
      for (int c = 0; c < kOC; c += 16) {
        uint32_t ov[16];
        tmem_ld_32x32b_x16(tO + lane_off + chh * kOC + c, ov);
        tmem_ld_wait_regs(ov);
#pragma unroll
        for (int j = 0; j < 16; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * alpha);
        tmem_st_32x32b_x16(tO + lane_off + chh * kOC + c, ov);
      }
      tmem_st_wait();
      l *= alpha;
    }
    if (refresh) m = mt;
    // P = exp2(S c2 - m) -> bf16 (smem K-major SW128 rows, or TMEM over S_t with PT), partial row sum
    const float mneg = -m;
    float rs4[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pk[PT ? kNC * 8 : 1];
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      float pv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float e = ex2_approx(fmaf(__uint_as_float(sr[c][j]), c2, mneg));
        pv[j] = (!need_mask || kbase + c * 16 + j <= qpos) ? e : 0.f;
        rs4[j & 3] += pv[j];
      }
      if constexpr (PT) {
#pragma unroll
        for (int j = 0; j < 8; ++j) pk[c * 8 + j] = pack_bf16x2(pv[2 * j], pv[2 * j + 1]);
      } else {
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8) {
          const int chunk = chunk0 + c * 2 + h8;  // 16-B chunk (8 keys) within the 128-B row
          uint4 w;
          w.x = pack_bf16x2(pv[h8 * 8 + 0], pv[h8 * 8 + 1]);
          w.y = pack_bf16x2(pv[h8 * 8 + 2], pv[h8 * 8 + 3]);
          w.z = pack_bf16x2(pv[h8 * 8 + 4], pv[h8 * 8 + 5]);
          w.w = pack_bf16x2(pv[h8 * 8 + 6], pv[h8 * 8 + 7]);
          *reinterpret_cast<uint4*>(prow + ((chunk ^ (r & 7)) << 4)) = w;
        }
      }
    }
    l += (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
    if constexpr (PT) {  // this half's 64 keys -> 32 packed columns at the start of its S columns
#pragma unroll
      for (int q = 0; q < kNC / 2; ++q)
        tmem_st_32x32b_x16(tS(sb) + lane_off + c_key0 + q * 16, *reinterpret_cast<const uint32_t(*)[16]>(&pk[q * 16]));
      tmem_st_wait();
      if (warp == 0 && t > 0) {  // V_{t-1} consumed by PV_{t-1} (also orders S_{t+2} after PV_{t-1})
        mbar_wait(o_done, (g - 1) & 1);
        tc_fence_after();
        if (t + 1 < ntiles) load_tile(t + 1, (g + 1) & 1, true);
      }
    } else {
      fence_proxy_async_shared();  // P (generic-proxy stores) -> visible to the tensor core
    }
    tc_fence_before();
    __syncthreads();  // P complete; S_buf reads, O rescales and red[] reads done
    if (tr) a.trace[t * 8 + 3] = globaltimer_ns();
    if (warp == 0) {  // O += P_t V_t  (TMEM accumulate)
      if (L::kVdb) mbar_wait(&v_full[buf], (g >> 1) & 1);
      else mbar_wait(&v_full[0], g & 1);
      tc_fence_after();
      const uint32_t pa = smem_u32(sP), vb = smem_u32(sV + (L::kVdb ? buf : 0) * L::kKV);
      if (PT && BK == 128 && a.mma8) {  // 8 k16 steps in one asm block; V descriptor + 2048 B per step
        umma8_ts(tO, tS(sb), make_desc_mn_sw128(vb, BK * 128, 1024), 2048 >> 4, idesc_o, t > 0 ? 1u : 0u);
      } else
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        const uint64_t bdesc = make_desc_mn_sw128(vb + k * 2048, BK * 128, 1024);
        if constexpr (PT)  // keys 16k..: column half k/4, packed columns 8(k mod 4)..
          umma_f16_ts_warp(tO, tS(sb) + (k >> 2) * 64 + (k & 3) * 8, bdesc, idesc_o, (t > 0 || k > 0) ? 1u : 0u);
        else
          umma_f16_ss_warp(tO, make_desc_k_sw128(pa + (k >> 2) * (kPBQ * 128) + (k & 3) * 32), bdesc, idesc_o,
                           (t > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit_warp(o_done);
    }
  }
  mbar_wait(o_done, (g0 + ntiles - 1) & 1);
  tc_fence_after();
  if (tr0 && n_done == 0) a.trace[255] = globaltimer_ns();
  red[chh * kPBQ + r] = l;
  named_bar_sync(1, 256);
  const float l_row = l + red[(chh ^ 1) * kPBQ + r];
  const float inv = 1.f / l_row;

  if (ksplit > 1) {
    // key split: unnormalised O half-row + (m, l) of this key range, then the pair's last CTA merges
    const int pq = qh * ntq + qt;
    const size_t prow = (static_cast<size_t>(pq) * ksplit + ks) * kPBQ + r;
    // O partial layout [pair][range][head_dim / 4][128 rows] float4: a warp's 32 rows of one
    // 4-dim group are 512 contiguous bytes (coalesced writes here and reads in the merge)
    float4* po4 = reinterpret_cast<float4*>(a.part_o) + (static_cast<size_t>(pq) * ksplit + ks) * (HD / 4) * kPBQ;
#pragma unroll
    for (int c = 0; c < kOC; c += 16) {
      uint32_t ov[16];
      tmem_ld_32x32b_x16(tO + lane_off + chh * kOC + c, ov);
      tmem_ld_wait_regs(ov);
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        __stcg(po4 + ((chh * kOC + c + j) >> 2) * kPBQ + r,
               make_float4(__uint_as_float(ov[j]), __uint_as_float(ov[j + 1]), __uint_as_float(ov[j + 2]),
                           __uint_as_float(ov[j + 3])));
    }
    if (chh == 0) __stcg(reinterpret_cast<float2*>(a.part_ml + 2 * prow), make_float2(m, l_row));
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(a.counters + pq, 1);
      s_merge = old == ksplit - 1;
      if (s_merge) a.counters[pq] = 0;  // re-arm for the next launch
    }
    __syncthreads();
    if (s_merge && q0 + r < p) {
      __threadfence();
      const size_t row0 = static_cast<size_t>(pq) * ksplit * kPBQ + r;  // + i * kPBQ per range
      // ksplit <= kMaxKsplit (host): every range's (m, l) and O loads are issued before they are used
      float mi[kMaxKsplit], li[kMaxKsplit], wi[kMaxKsplit];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kMaxKsplit; ++i) {
        const float2 ml = i < ksplit ? __ldcg(reinterpret_cast<const float2*>(a.part_ml + 2 * (row0 + i * kPBQ)))
                                     : make_float2(-INFINITY, 0.f);
        mi[i] = ml.x;
        li[i] = ml.y;
        mx = fmaxf(mx, ml.x);
      }
      float lsum = 0.f;
#pragma unroll
      for (int i = 0; i < kMaxKsplit; ++i) {
        wi[i] = mi[i] == -INFINITY ? 0.f : exp2f(mi[i] - mx);  // ranges past ksplit: m = -inf
        lsum = fmaf(wi[i], li[i], lsum);
      }
      const float linv = 1.f / lsum;
      __nv_bfloat16* dst = a.out + static_cast<size_t>(a.q_row0 + q0 + r) * a.out_ld + qh * HD + chh * kOC;
#pragma unroll 2
      for (int c = 0; c < kOC; c += 8) {
        float4 x[kMaxKsplit][2];
#pragma unroll
        for (int i = 0; i < kMaxKsplit; ++i) {
          const float4* src = reinterpret_cast<const float4*>(a.part_o) +
                              (static_cast<size_t>(pq) * ksplit + i) * (HD / 4) * kPBQ +
                              ((chh * kOC + c) >> 2) * kPBQ + r;
          x[i][0] = i < ksplit ? __ldcg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
          x[i][1] = i < ksplit ? __ldcg(src + kPBQ) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < kMaxKsplit; ++i) {
          const float w = wi[i] * linv;
          acc[0] = fmaf(x[i][0].x, w, acc[0]); acc[1] = fmaf(x[i][0].y, w, acc[1]);
          acc[2] = fmaf(x[i][0].z, w, acc[2]); acc[3] = fmaf(x[i][0].w, w, acc[3]);
          acc[4] = fmaf(x[i][1].x, w, acc[4]); acc[5] = fmaf(x[i][1].y, w, acc[5]);
          acc[6] = fmaf(x[i][1].z, w, acc[6]); acc[7] = fmaf(x[i][1].w, w, acc[7]);
        }
        uint4 o4;
        o4.x = pack_bf16x2(acc[0], acc[1]);
        o4.y = pack_bf16x2(acc[2], acc[3]);
        o4.z = pack_bf16x2(acc[4], acc[5]);
        o4.w = pack_bf16x2(acc[6], acc[7]);
        *reinterpret_cast<uint4*>(dst + c) = o4;
      }
    }
  } else
  // O rows (bf16): this warp's half of the row's dims; rows past the chunk are not written
  {
    __nv_bfloat16* dst = a.out + static_cast<size_t>(a.q_row0 + q0 + r) * a.out_ld + qh * HD + chh * kOC;
    const bool valid = q0 + r < p;
#pragma unroll
    for (int c = 0; c < kOC; c += 16) {
      uint32_t ov[16];
      tmem_ld_32x32b_x16(tO + lane_off + chh * kOC + c, ov);
      tmem_ld_wait_regs(ov);
      if (valid) {
#pragma unroll
        for (int h8 = 0; h8 < 16; h8 += 8) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(ov[h8 + 0]) * inv, __uint_as_float(ov[h8 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(ov[h8 + 2]) * inv, __uint_as_float(ov[h8 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(ov[h8 + 4]) * inv, __uint_as_float(ov[h8 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(ov[h8 + 6]) * inv, __uint_as_float(ov[h8 + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c + h8) = w;
        }
      }
    }
  }
  g0 += ntiles;
  tc_fence_before();
  __syncthreads();  // O / red / Q / K,V buffers free for the next item
  tc_fence_after();
  }  // item loop
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, L::kTmemCols);
  }
  if (a.done_flag) {  // the grid's last CTA to finish publishes completion (O GEMM X dependency)
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int total = static_cast<int>(gridDim.x * gridDim.y * gridDim.z);
      const int old = atomicAdd(a.done_cnt, 1);
      if (old == total - 1) {
        *a.done_cnt = 0;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.done_flag), "r"(a.epoch) : "memory");
      }
    }
  }
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 384) a.trace[257 + 2 * blockIdx.x] = globaltimer_ns();
  if (a.span_end && threadIdx.x == 0) atomicMax(a.span_end, globaltimer_ns());
}

template <int HD>
cudaError_t launch_decode_hd(const DecodeAttnArgs& a, const CUtensorMap& mk, const CUtensorMap& mv, cudaStream_t st) {
  const size_t smem = decode_smem_bytes(HD, a.block_size, a.stages, 1);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(decode_attn_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    prefer_max_smem(decode_attn_mma<HD>);
    configured = true;
  }
  dim3 grid(a.d, a.n_kv_local, a.splits);
  if (a.no_pdl)
    decode_attn_mma<HD><<<grid, 160, smem, st>>>(mk, mv, a);
  else
    launch_pdl(decode_attn_mma<HD>, grid, dim3(160), smem, st, mk, mv, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1) return e;
  launch_pdl(decode_combine_kernel, dim3(a.d, a.n_q_local), dim3(128), 0, st, a, HD);
  return cudaGetLastError();
}

}  // namespace

size_t decode_smem_bytes(int head_dim, int block_size, int stages, int /*G*/) {
  const size_t ring = static_cast<size_t>(stages) * 2 * block_size * head_dim * 2;
  const size_t merge = (128 + 64 * static_cast<size_t>(head_dim)) * 4;
  return std::max(ring, merge) + 16 * stages + 1024 + 64;
}

bool make_tmap_kv(CUtensorMap* map, const void* pool, long long rows, int head_dim, int block_size) {
  // 2D view [rows = num_blocks * n_kv * block_size][head_dim], 64-column boxes of block_size rows, SW128
  return make_tmap_bf16(map, pool, static_cast<uint64_t>(rows), head_dim, head_dim, block_size);
}

cudaError_t launch_decode_attention(const DecodeAttnArgs& a, const CUtensorMap& mk, const CUtensorMap& mv,
                                    cudaStream_t st) {
  if (a.d == 0) return cudaSuccess;
  if (a.n_q_local / a.n_kv_local > 16) return cudaErrorInvalidValue;
  if (a.head_dim == 128) return launch_decode_hd<128>(a, mk, mv, st);
  if (a.head_dim == 64) return launch_decode_hd<64>(a, mk, mv, st);
  return cudaErrorInvalidValue;
}

template <int HD, int BK, bool PT = false>
cudaError_t launch_prefill_tc(const PrefillAttnArgs& a, const CUtensorMap& mq, const CUtensorMap& mk,
                              const CUtensorMap& mv, cudaStream_t st) {
  using L = PtcSmem<HD, BK, PT>;
  static bool configured = false;
  if (!configured) {
    prefer_max_smem(prefill_attn_tc<HD, BK, PT>);
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_tc<HD, BK, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(L::kTotal));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int items = (a.p + kPBQ - 1) / kPBQ * a.n_q_local * std::max(1, a.ksplit);
  static const int cap = getenv("SARATHI_PREFILL_CTAS") ? atoi(getenv("SARATHI_PREFILL_CTAS")) : 0;  // experiment
  const int ctas = cap > 0 ? std::min(cap, items) : items;
  static const bool mma8 = !(getenv("SARATHI_ATTN_MMA8") && atoi(getenv("SARATHI_ATTN_MMA8")) == 0);
  PrefillAttnArgs a8 = a;
  a8.mma8 = mma8 ? 1 : 0;
  if (a.pdl)
    launch_pdl(prefill_attn_tc<HD, BK, PT>, dim3(ctas), dim3(256), L::kTotal, st, mq, mk, mv, a8);
  else
    prefill_attn_tc<HD, BK, PT><<<ctas, 256, L::kTotal, st>>>(mq, mk, mv, a8);
  return cudaGetLastError();
}

cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, const CUtensorMap* qmap, const CUtensorMap* kmap,
                                     const CUtensorMap* vmap, cudaStream_t st) {
  if (a.p == 0) return cudaSuccess;
  if (!qmap || !kmap || !vmap || 128 % a.block_size) return cudaErrorInvalidValue;  // alloc_kv: bs | 128
  // 128-key tiles; SARATHI_PREFILL_BK=64 selects the narrow tile (2 CTAs or a CTA + decode CTAs per
  // SM).  Measured: TP-1 step unchanged, TP-8 rank shapes 2-4 % slower, so not the default.
  static const bool narrow = getenv("SARATHI_PREFILL_BK") && atoi(getenv("SARATHI_PREFILL_BK")) == 64;
  const bool bk128 = a.block_size == 128 || !narrow;
  // P in TMEM (default); SARATHI_PREFILL_PT=0 selects the smem P image
  static const bool pt = !(getenv("SARATHI_PREFILL_PT") && atoi(getenv("SARATHI_PREFILL_PT")) == 0);
  if (a.head_dim == 128)
    return !bk128 ? launch_prefill_tc<128, 64>(a, *qmap, *kmap, *vmap, st)
           : pt   ? launch_prefill_tc<128, 128, true>(a, *qmap, *kmap, *vmap, st)
                  : launch_prefill_tc<128, 128>(a, *qmap, *kmap, *vmap, st);
  if (a.head_dim == 64)
    return !bk128 ? launch_prefill_tc<64, 64>(a, *qmap, *kmap, *vmap, st)
           : pt   ? launch_prefill_tc<64, 128, true>(a, *qmap, *kmap, *vmap, st)
                  : launch_prefill_tc<64, 128>(a, *qmap, *kmap, *vmap, st);
  return cudaErrorInvalidValue;
}

}  // namespace sarathi

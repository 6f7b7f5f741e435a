// tcgen05 / TMEM / TMA bf16 GEMM for the hybrid-batch linears (preproj, postproj, ffn_ln1,
// ffn_ln2 and the LM head; PAPER.md L214-221 Table table:tensor:shapes, §2.1).
//
// Decode-maximal batching fuses all p + d tokens of a hybrid batch into ONE matmul per linear so
// every weight byte is fetched once for both kinds of token (§4.3).  With
// T = p + d <= 512 tokens per batch the sm_100a mapping is "swap-AB":
//     D[m, t] = sum_k W[m, k] * X[t, k]     UMMA M = 128 weight rows, N = all tokens (<= 256 per
//                                           instruction, two instructions when T > 256), K = 16
// so each weight byte is streamed from HBM exactly once while the small token matrix stays in L2.
//
// Persistent stream-K: grid = #SMs (1 CTA per SM); the (tile, k-block) iteration space is cut
// into equal contiguous ranges, one per CTA, so every SM does the same amount of MMA work whatever
// the number of 128-row tiles (QKV 120, O 40, gate/up 216, down 40, LM head 250 at LLaMA-13B).
// A tile covered by several CTAs is reduced deterministically: each contributor writes an fp32
// partial into its slot, the last to arrive (atomic counter) sums the slots in order and runs the
// fused epilogue.  Warp roles (320 threads):
//   warp 0      TMA producer: W tile [128 x 64] (evict_first) + X tile [bn x 64] (evict_last),
//               128B swizzle, S-stage smem ring (full/empty mbarriers), runs across segments
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; tcgen05.commit frees stages and
//               signals the epilogue per segment; TMEM double-buffered when bn <= 256
//   warps 2..9  epilogue straight from TMEM (tcgen05.ld 32x32b.x16; two warps per lane quarter,
//               alternate 16-token chunks): residual add, SiLU*up,
//               GELU, RoPE + paged KV append, bf16/fp32 stores, or the stream-K partial
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "host_sched.hpp"

#include <algorithm>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace sarathi {

namespace {


struct KParams {
  int M, N, KB;
  int bn, n_mma;          // tokens per tile; UMMAs per k-step (bn / n_mma tokens each, <= 256)
  int pm_tiles, n_tiles;  // 256-row pair tiles, token tiles
  long long units;        // stream-K units = sk_tiles * KB (the first sk_tiles tiles are split)
  int ctas;               // number of CTA PAIRS (grid = 2 * ctas)
  int sk_tiles;           // tiles processed stream-K (first), split across all pairs
  int dp_per_pair;        // whole tiles per pair processed after the stream-K part
  int dp_extra;           // pairs [0, dp_extra) take one more whole tile
  int half_items;         // pairs [0, half_items) then take one token half of a remainder tile
  int tiles;              // total pair-tiles = pm_tiles * n_tiles
  int stages;
  int nbuf;               // TMEM accumulator buffers (2 if bn <= 256)
  int max_slots;          // partial slots per tile
  int red_partials;       // split tiles accumulate in ONE zeroed fp32 slot by red.add (many contributors)
  int atomic;             // residual add: every contributor red.adds its partial (else slots, deterministic)
  uint32_t tmem_cols;
  uint32_t ring_bytes;
  int n0, n1;             // tokens of UMMA 0 / 1 per k-step (n_mma == 2: equal halves, or 256 + tail)
  int ts;                 // A (weights) staged in TMEM by tcgen05.cp at column kTsCol: the second UMMA of
                          // a k-step does not re-read A from shared memory
};
constexpr int kTsCol = 480;  // 4 k16 slices x 8 columns of the A operand (one k-block)


// X-flag wait (EpiParams::xflag): relaxed spin, one acquire fence, then order the async proxy (TMA)
// after it; a lost flag traps instead of hanging the GPU
SARATHI_DEVICE void xflag_wait(const unsigned* f, unsigned epoch) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  if (static_cast<int>(v - epoch) < 0) {
    const unsigned long long t0 = globaltimer_ns();
    do {
      __nanosleep(64);
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (globaltimer_ns() - t0 > 4000000000ull) __trap();
    } while (static_cast<int>(v - epoch) < 0);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

SARATHI_DEVICE long long unit_begin(int c, const KParams& p) {
  return (static_cast<long long>(c) * p.units) / p.ctas;
}
// CTA pair owning stream-K unit u under the balanced partition above (units > 0).
SARATHI_DEVICE int cta_of(long long u, const KParams& p) {
  return static_cast<int>(((u + 1) * p.ctas - 1) / p.units);
}

// Work of one CTA pair: first its stream-K range of units over the split tiles [0, sk_tiles) (so
// their reductions overlap later work), then dp_per_pair whole tiles (reduction-free epilogues).
// Finally (p.half_items > 0) one token-half item: the tiles % P remainder tiles are not split over
// K (partials + a reduction pass) but over their two UMMA token halves, one half per pair.
struct SegIter {
  long long u, u_end;
  int dp_t, dp_end;
  int hi;    // this pair's token-half item (-1: none or done)
  int half;  // of the segment returned last: -1 whole tile / k-range, else the token half (UMMA 0 / 1)
  SARATHI_DEVICE void init(const KParams& p, int pair) {
    u = unit_begin(pair, p);
    u_end = unit_begin(pair + 1, p);
    dp_t = p.sk_tiles + pair * p.dp_per_pair + min(pair, p.dp_extra);
    dp_end = min(p.tiles - p.half_items / 2, dp_t + p.dp_per_pair + (pair < p.dp_extra ? 1 : 0));
    hi = pair < p.half_items ? pair : -1;
    half = -1;
  }
  // next segment: tile, k-block range [kb0, kb1); false when done
  SARATHI_DEVICE bool next(const KParams& p, int& tile, int& kb0, int& kb1) {
    half = -1;
    if (u < u_end) {
      tile = static_cast<int>(u / p.KB);
      kb0 = static_cast<int>(u % p.KB);
      kb1 = static_cast<int>(min(static_cast<long long>(p.KB), kb0 + (u_end - u)));
      u += kb1 - kb0;
      return true;
    }
    if (dp_t < dp_end) {
      tile = dp_t++;
      kb0 = 0;
      kb1 = p.KB;
      return true;
    }
    if (hi >= 0) {
      tile = p.tiles - p.half_items / 2 + (hi >> 1);
      half = hi & 1;
      hi = -1;
      kb0 = 0;
      kb1 = p.KB;
      return true;
    }
    return false;
  }
};


// RMSNorm (reading O-8, Table 1 "ln" rows) of rows r = blockIdx.x, blockIdx.x + grid, ...
// of h (fp32 [T][H]) into out (bf16 [T][H]: x * rsqrt(mean x^2 + eps) * g) by the whole CTA (kThr
// threads, named barrier 3); up to kMaxRows rows are normalised together (all their loads in flight,
// one reduction round).  `red` = kMaxRows x 16 floats of scratch shared memory.  The per-row sum is
// reduced in a fixed order (warp shuffles, then warps in index order): deterministic.
template <int kThr>
SARATHI_DEVICE void norm_rows(const float* h, const __nv_bfloat16* g, __nv_bfloat16* xo, int T, int H, float eps,
                              float* red) {
  constexpr int kMaxRows = 4;
  const int tid = threadIdx.x;
  const uint32_t warp = tid >> 5, lane = tid & 31;
  for (int r0 = blockIdx.x; r0 < T; r0 += kMaxRows * gridDim.x) {
    float4 v[kMaxRows][4];
    float ss[kMaxRows];
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) {
      const int r = r0 + j * gridDim.x;
      ss[j] = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = (c * kThr + tid) * 4;
        v[j][c] = (r < T && i < H) ? __ldcg(reinterpret_cast<const float4*>(h + static_cast<size_t>(r) * H + i))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) {
      const int r = r0 + j * gridDim.x;
#pragma unroll
      for (int c = 0; c < 4; ++c) ss[j] += v[j][c].x * v[j][c].x + v[j][c].y * v[j][c].y + v[j][c].z * v[j][c].z + v[j][c].w * v[j][c].w;
      if (r < T)
        for (int i = (4 * kThr + tid) * 4; i < H; i += kThr * 4) {  // H > 4 * 4 * threads
          const float4 w = __ldcg(reinterpret_cast<const float4*>(h + static_cast<size_t>(r) * H + i));
          ss[j] += w.x * w.x + w.y * w.y + w.z * w.z + w.w * w.w;
        }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], off);
      if (lane == 0) red[j * 16 + warp] = ss[j];
    }
    named_bar_sync(3, kThr);
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) {
      const int r = r0 + j * gridDim.x;
      if (r >= T) break;
      float tot = 0.f;
      for (int w = 0; w < kThr / 32; ++w) tot += red[j * 16 + w];  // warp order: deterministic
      const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
      auto put = [&](int i, float4 w) {
        const uint2 graw = *reinterpret_cast<const uint2*>(g + i);
        const float2 g01 = unpack_bf16x2(graw.x), g23 = unpack_bf16x2(graw.y);
        uint2 pk;
        pk.x = pack_bf16x2(w.x * inv * g01.x, w.y * inv * g01.y);
        pk.y = pack_bf16x2(w.z * inv * g23.x, w.w * inv * g23.y);
        *reinterpret_cast<uint2*>(xo + static_cast<size_t>(r) * H + i) = pk;
      };
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = (c * kThr + tid) * 4;
        if (i < H) put(i, v[j][c]);
      }
      for (int i = (4 * kThr + tid) * 4; i < H; i += kThr * 4)
        put(i, __ldcg(reinterpret_cast<const float4*>(h + static_cast<size_t>(r) * H + i)));
    }
    named_bar_sync(3, kThr);  // (red is rewritten by the next group of rows)
  }
}

template <int NEH, int MODE, bool DBG>
__global__ void __launch_bounds__(threads_of<NEH>(), 1)
    gemm_bf16_pair(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX,
                   const __grid_constant__ CUtensorMap mapX2, const KParams p,
                   const EpiParams ep) {
  constexpr int kEpiThreads = 128 * NEH;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base derived by pointer arithmetic from the __shared__ array (not an integer
  // round trip), so every pointer below stays in the shared address space (STS/LDS, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t b_bytes = static_cast<uint32_t>(p.bn / 2) * kBK * 2;  // this CTA's half of the tokens
  const uint32_t stage_bytes = kABytes + b_bytes;
  float* stage_buf = reinterpret_cast<float*>(smem + p.ring_bytes);    // [8 warps][16 x 32] transpose
  int* s_pos = reinterpret_cast<int*>(stage_buf + 4 * NEH * kStageFloats);  // [bn]
  int* s_slot = s_pos + p.bn;                                          // [bn]
  int* s_consec = s_slot + p.bn;                                       // [32] chunk has consecutive positions
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_consec + 32);         // 8-B aligned (bn is a multiple of 16)
  uint64_t* full = bars;                // local: this CTA's W + X bytes landed
  uint64_t* pfull = full + p.stages;    // leader only: the peer's stage landed (relayed)
  uint64_t* empty = pfull + p.stages;
  uint64_t* tfull = empty + p.stages;   // [2]
  uint64_t* tempty = tfull + 2;         // [3] (leader's are the ones waited on)
  uint32_t* holder = reinterpret_cast<uint32_t*>(tempty + 3);
  __shared__ int s_last;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();   // 0 = leader (issues the pair MMAs)
  griddep_launch_dependents();
  if (ep.span_start && threadIdx.x == 0) atomicMin(ep.span_start, globaltimer_ns());
  const int pair = blockIdx.x >> 1;
  // debug trace: CTA pair (dbg >> 8) records its timeline (tb = 0 / 1 for its two CTAs)
  const int tb = static_cast<int>(blockIdx.x) - 2 * (ep.dbg >> 8);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&pfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&tfull[b], 1);
    for (int b = 0; b < 3; ++b) mbar_init(&tempty[b], 8 * NEH);  // 4*NEH epilogue warps x 2 CTAs
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapW);
    tma_prefetch_desc(&mapX);
    if (p.n0 != p.n1) tma_prefetch_desc(&mapX2);
  }
  if (warp == 1) tmem_alloc_pair(holder, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const int ni = p.bn / p.n_mma;  // tokens per UMMA (multiple of 16, <= 256)
  // TMEM slot ring (two UMMAs per k-step, 3 * ni <= 512): segment s accumulates into slots
  // (2s mod 3, 2s+1 mod 3) of ni columns, so segment s+1 only needs the first half of segment s's
  // accumulator drained (its other slot was freed a segment earlier) and the next mainloop overlaps
  // most of the epilogue.  Otherwise: two 256-column buffers (bn <= 256) or one.
  // uneven split (n0 = 256 + a 16..240-token tail n1, single accumulator): one full-width UMMA plus
  // a narrow one instead of two halves, for single-segment plans (no epilogue overlap to keep)
  const bool ring = p.n_mma == 2 && p.n0 == p.n1 && 3 * ni <= 512;
  if (ep.norm_h) {
    constexpr int kThr = 64 + 128 * NEH;  // threads per CTA
    // fused RMSNorm prologue: the producer first issues its first ring of W tiles (they do not
    // depend on the predecessor), then every thread waits for the grid dependency, normalises its
    // CTA's rows, and the grid meets at a barrier before the first X load
    if (warp == 0) {
      SegIter it0;
      it0.init(p, pair);
      int tile, kb0, kb1;
      if (it0.next(p, tile, kb0, kb1)) {
        const uint32_t tx = 2 * stage_bytes - (it0.half >= 0 ? 2u * (p.n1 / 2) * kBK * 2 : 0u);
        const int npre0 = min(p.stages, kb1 - kb0);
        const int pt = tile / p.n_tiles;
        const int wrow0 = ((pt * 2 + static_cast<int>(rank)) * p.KB + kb0) * kWRowsPerTile;
        for (int j = 0; j < npre0; ++j) {
          if (rank == 0) mbar_arrive_expect_tx_warp(&full[j], tx);
          tma_load_2d_pair_warp(smem + static_cast<size_t>(j) * stage_bytes, &mapW, &full[j], 0,
                                wrow0 + j * kWRowsPerTile, policy_evict_first());
        }
      }
    }
    griddep_wait();
    norm_rows<64 + 128 * NEH>(ep.norm_h, static_cast<const __nv_bfloat16*>(ep.norm_g),
                              static_cast<__nv_bfloat16*>(ep.norm_out), ep.norm_T, ep.norm_H, ep.norm_eps, stage_buf);
    // grid barrier: every CTA's rows written (and visible to the async proxy) before any X load
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    named_bar_sync(3, kThr);
    if (threadIdx.x == 0) {
      atomicAdd(ep.norm_ctr, 1u);
      xflag_wait(ep.norm_ctr, ep.norm_target);
    }
    named_bar_sync(3, kThr);
  } else {
    // the producer waits after prefetching its first W tiles; with X flags (ep.xflag) only the
    // epilogue waits for the predecessor grid
    if (warp >= 2 || (warp == 1 && !ep.xflag)) griddep_wait();
  }

  if (warp == 0) {
    // ---------------- TMA producer (whole warp, warp-uniform; one elected lane issues) ----------------
    {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // incremental (k-block, stage, phase) counters inside a segment: no division in the hot loop
      const uint32_t tx = 2 * (stage_bytes - ((DBG && (ep.dbg & 1)) ? b_bytes : 0) - ((DBG && (ep.dbg & 2)) ? kABytes : 0));
      // a token-half item loads only its UMMA's half of the tokens
      const uint32_t txh = (DBG && (ep.dbg & 1)) ? tx : tx - 2u * (p.n1 / 2) * kBK * 2;
      int s = 0;
      uint32_t ph = 0;
      long long i = 0;
      SegIter it;
      it.init(p, pair);
      int tile, kb0, kb1;
      // PDL: weights do not depend on the previous kernel, so the first ring's W tiles are fetched
      // before the grid-dependency wait (overlapping the predecessor's tail); X loads come after it
      int npre = 0;
      if (ep.norm_h) {  // the prologue issued the first ring of W tiles already
        SegIter it0 = it;
        if (it0.next(p, tile, kb0, kb1)) npre = min(p.stages, kb1 - kb0);
      } else {
        SegIter it0 = it;
        if (it0.next(p, tile, kb0, kb1)) {
          npre = min(p.stages, kb1 - kb0);
          const int pt = tile / p.n_tiles;
          const int wrow0 = ((pt * 2 + static_cast<int>(rank)) * p.KB + kb0) * kWRowsPerTile;
          for (int j = 0; j < npre; ++j) {
            uint8_t* a = smem + static_cast<size_t>(j) * stage_bytes;
            if (rank == 0) mbar_arrive_expect_tx_warp(&full[j], it0.half >= 0 ? txh : tx);
            if (!(DBG && (ep.dbg & 2))) tma_load_2d_pair_warp(a, &mapW, &full[j], 0, wrow0 + j * kWRowsPerTile, pol_w);
          }
        }
      }
      if (ep.norm_h) {
        // grid dependency and X (this kernel's own prologue) already waited for
      } else if (!ep.xflag) {
        griddep_wait();
      } else if (ep.xflag2) {
        xflag_wait(ep.xflag2, ep.xepoch);
      }
      int have_lo = 0, have = -1;  // X flags [have_lo, have] already acquired (ep.xflag)
      while (it.next(p, tile, kb0, kb1)) {
        const int pt = tile / p.n_tiles, nt = tile % p.n_tiles;
        int wrow = ((pt * 2 + static_cast<int>(rank)) * p.KB + kb0) * kWRowsPerTile;  // row in the 512-B view
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          uint8_t* a = smem + static_cast<size_t>(s) * stage_bytes;
          uint8_t* b = a + kABytes;
          if (i >= npre) {
            mbar_wait(&empty[s], ph ^ 1);
            // both CTAs' bytes are counted on the leader's full[s] (pair TMA)
            if (rank == 0) mbar_arrive_expect_tx_warp(&full[s], it.half >= 0 ? txh : tx);
            // W tile: the contiguous 16 KB pre-swizzled tile as 32 rows x 512 B (unswizzled map)
            if (!(DBG && (ep.dbg & 2))) tma_load_2d_pair_warp(a, &mapW, &full[s], 0, wrow, pol_w);
          }
          if (ep.xflag) {
            const int need = (kb * kBK) / ep.xflag_cols;
            if (need < have_lo || need > have) {
              // warp-wide relaxed scan of the next 32 flags, block on the first unready one only
              have_lo = need;
              while (true) {
                const int q = need + static_cast<int>(lane);
                unsigned v = 0xFFFFFFFFu;
                if (q < ep.xflag_n) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ep.xflag + q) : "memory");
                const bool ok = q >= ep.xflag_n || static_cast<int>(v - ep.xepoch) >= 0;
                const unsigned bad = __ballot_sync(0xffffffffu, !ok);
                const int nready = bad ? __ffs(bad) - 1 : 32;
                if (nready > 0) {
                  have = need + nready - 1;
                  break;
                }
                xflag_wait(ep.xflag + need, ep.xepoch);
              }
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
          }
          if (DBG && (ep.dbg & 1)) {
          } else if (it.half >= 0) {  // token-half item (n0 == n1): UMMA `half`'s tokens into the first B slot
            tma_load_2d_pair_warp(b, &mapX, &full[s], kb * kBK, nt * p.bn + it.half * p.n0 + static_cast<int>(rank) * (p.n0 / 2),
                                  pol_x);
          } else {
            tma_load_2d_pair_warp(b, &mapX, &full[s], kb * kBK, nt * p.bn + static_cast<int>(rank) * (p.n0 / 2), pol_x);
            if (p.n_mma == 2)
              tma_load_2d_pair_warp(b + (p.n0 / 2) * kBK * 2, p.n0 == p.n1 ? &mapX : &mapX2, &full[s], kb * kBK,
                                    nt * p.bn + p.n0 + static_cast<int>(rank) * (p.n1 / 2), pol_x);
          }
          if ((DBG ? ep.trace : nullptr) && tb < 2 && i < 256 && lane == 0) (DBG ? ep.trace : nullptr)[tb * 1024 + i] = globaltimer_ns();
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
          wrow += kWRowsPerTile;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader, lane 0) / stage relay (peer) ----------------
    if (rank == 0) {
      // k-block issue from one asm block for two UMMAs per k-step and for narrow single UMMAs (issue-
      // paced); single wide UMMAs (N >= 192) keep the per-UMMA statements, measured 1-3 % faster at
      // T = 256 (QKV 46.4 vs 47.9 us, down 39.5 vs 40.9; profiles/r02_t256_kbasm.txt).
      // SARATHI_GEMM_KBASM=0: the per-UMMA path everywhere.
      const bool kblock_asm = ep.kbasm && (p.n_mma == 2 || p.n0 < 192);
      const uint32_t idesc = make_idesc_bf16_f32(2 * kBM, p.n0);
      const uint32_t idesc1 = make_idesc_bf16_f32(2 * kBM, p.n1);
      int i = 0, seg = 0, s = 0;
      uint32_t ph = 0;
      SegIter it;
      it.init(p, pair);
      int tile, kb0, kb1;
      int uses[3] = {0, 0, 0};
      int rs = 0;  // ring slots taken so far (a whole tile takes two, a token-half item one)
      while (it.next(p, tile, kb0, kb1)) {
        const int buf = seg % p.nbuf;
        const uint32_t use = seg / p.nbuf;
        const bool hseg = it.half >= 0;
        uint32_t d0, d1;
        int tb_idx;  // tfull barrier of this segment
        if (ring) {
          const int sa = rs % 3, sb = (rs + 1) % 3;
          rs += hseg ? 1 : 2;
          for (int k : {sa, sb}) {  // both CTAs' epilogues drained the slot's previous use
            if (hseg && k == sb) continue;
            if (uses[k]) mbar_wait_cluster(&tempty[k], (uses[k] - 1) & 1);
            ++uses[k];
          }
          d0 = tmem + sa * ni;
          d1 = tmem + sb * ni;
          tb_idx = seg & 1;
        } else {
          mbar_wait_cluster(&tempty[buf], (use & 1) ^ 1);  // both CTAs' epilogues drained it
          d0 = tmem + buf * 256;
          d1 = d0 + p.n0;
          tb_idx = buf;
        }
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if ((DBG ? ep.trace : nullptr) && tb == 0 && lane == 0 && i < 256) (DBG ? ep.trace : nullptr)[256 + i] = globaltimer_ns();
          {
            // warp-uniform issue (operands stay in uniform registers), one elected lane issues
            const uint32_t a = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
            const uint32_t b = a + kABytes;
            if (kblock_asm) {
              // the whole k-block in one asm block (one elect, descriptors advanced in registers)
              const uint32_t acc0 = kb != kb0 ? 1u : 0u;
              const uint32_t two = (p.n_mma == 2 && !hseg) ? 1u : 0u;
              if (p.ts)
                umma_kblock_ts_pair(d0, d1, tmem + kTsCol, make_desc_k_sw128(a), make_desc_k_sw128(b),
                                    make_desc_k_sw128(b + (p.n0 / 2) * 128), idesc, idesc1, acc0, two);
              else
                umma_kblock_ss_pair(d0, d1, make_desc_k_sw128(a), make_desc_k_sw128(b),
                                    make_desc_k_sw128(b + (p.n0 / 2) * 128), idesc, idesc1, acc0, two);
            } else if (p.ts) {
              const uint32_t at = tmem + kTsCol;
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
                tmem_cp_128x256b_pair_warp(at + k * 8, make_desc_k_sw128(a + k * 32));
                umma_f16_ts_pair_warp(d0, at + k * 8, make_desc_k_sw128(b + k * 32), idesc, acc);
                if (!hseg)
                  umma_f16_ts_pair_warp(d1, at + k * 8, make_desc_k_sw128(b + (p.n0 / 2) * 128 + k * 32), idesc1, acc);
              }
            } else {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
                umma_f16_ss_pair_warp(d0, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, acc);
                if (p.n_mma == 2 && !hseg)
                  umma_f16_ss_pair_warp(d1, make_desc_k_sw128(a + k * 32),
                                        make_desc_k_sw128(b + (p.n0 / 2) * 128 + k * 32), idesc1, acc);
              }
            }
            umma_commit_pair_mc_warp(&empty[s], 0x3);
            if (kb == kb1 - 1) umma_commit_pair_mc_warp(&tfull[tb_idx], 0x3);
          }
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        ++seg;
      }
    }
  } else {
    // ---------------- Epilogue (warps 2..9 of both CTAs) ----------------
    // NEH warps per TMEM lane quarter (warp & 3); warp `eh` of a quarter takes chunks eh, eh + NEH, ...
    const int et = threadIdx.x - 64;                        // 0..255
    const int ew = static_cast<int>(warp) - 2;              // 0..7
    const int eh = ew >> 2;
    const uint32_t quarter = warp & 3;                      // TMEM lane quarter of this warp
    float* sbuf = stage_buf + ew * kStageFloats;            // this warp's transpose buffer
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    const bool relaxed_rel = ep.relaxed_rel;  // SARATHI_GEMM_RELAXED=0: release.cluster arrives
    int seg = 0;
    int rs = 0;  // ring slots taken so far (as the MMA issuer counts them)
    const size_t tile_elems = static_cast<size_t>(p.bn) * kBM;
    constexpr bool rope_mode = MODE == EPI_QKV_ROPE;
    SegIter it;
    it.init(p, pair);
    int tile, kb0, kb1;
    while (it.next(p, tile, kb0, kb1)) {
      const int pt = tile / p.n_tiles, nt = tile % p.n_tiles;
      const int mt = pt * 2 + static_cast<int>(rank);       // this CTA's 128-row tile
      const int buf = seg % p.nbuf;
      const uint32_t use = seg / p.nbuf;
      const int tvalid = min(p.bn, p.N - nt * p.bn);
      // whole tiles and residual adds (red.add of every contributor's partial) emit straight from TMEM
      const bool direct = (kb0 == 0 && kb1 == p.KB) || (MODE == EPI_ADD_F32 && p.atomic);
      QkvLane ql{};
      if (rope_mode) ql = qkv_lane(ep, mt, quarter, lane);
      const int nchunks = (tvalid + 15) / 16;
      // accumulator column of chunk ch and the TMEM releases this warp owes (see `ring`)
      const int nA = ring ? ni / 16 : (1 << 30);
      const bool hseg = it.half >= 0;  // token-half item: chunks [c_lo, c_hi) in ONE ring slot
      const int sA = rs % 3, sB = (rs + 1) % 3;
      rs += hseg ? 1 : 2;
      const int c_lo = hseg ? it.half * nA : 0, c_hi = hseg ? min(c_lo + nA, nchunks) : nchunks;
      auto tcol = [&](int ch) -> uint32_t {
        if (!ring) return static_cast<uint32_t>(buf * 256 + ch * 16);
        if (hseg) return static_cast<uint32_t>(sA * ni + (ch - c_lo) * 16);
        return static_cast<uint32_t>(ch < nA ? sA * ni + ch * 16 : sB * ni + (ch - nA) * 16);
      };
      auto arrive_slot = [&](int k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (relaxed_rel)
            mbar_arrive_cluster_relaxed(tempty_leader + k * 8);
          else
            mbar_arrive_cluster(tempty_leader + k * 8);
        }
      };
      auto last_of = [&](int lim) {  // this warp's last chunk in [c_lo, lim) (-1 if none)
        if (lim <= c_lo + eh) return -1;
        return c_lo + eh + ((lim - 1 - c_lo - eh) / NEH) * NEH;
      };
      const int lastA = hseg ? -1 : last_of(min(nA, nchunks)), lastAll = last_of(c_hi);
      auto release_tmem = [&]() {  // everything this warp owes for the segment
        if (ring) {
          arrive_slot(sA);
          if (!hseg) arrive_slot(sB);
        } else {
          arrive_slot(buf);
        }
      };
      auto after_load = [&](int c) {  // chunk c's accumulator is in registers
        if (ring) {
          if (hseg) {
            if (c == lastAll) arrive_slot(sA);
          } else {
            if (c == lastA) arrive_slot(sA);
            if (c == lastAll) arrive_slot(sB);  // (with A when this warp has no half-B chunk)
          }
        } else if (c == lastAll) {
          arrive_slot(buf);
        }
      };
      if (rope_mode) {  // stage per-token metadata for the fused KV append
        named_bar_sync(2, kEpiThreads);
        for (int t = et; t < tvalid; t += kEpiThreads) {
          s_pos[t] = __ldg(ep.pos + nt * p.bn + t);
          const int sl = __ldg(ep.slot + nt * p.bn + t);
          // paged-cache row of (slot, kv head 0): [block][n_kv][bs] -> (sl/bs)*n_kv*bs + sl%bs
          s_slot[t] = (sl / ep.block_size) * ep.n_kv_local * ep.block_size + sl % ep.block_size;
        }
        named_bar_sync(2, kEpiThreads);
        if (et < (tvalid + 15) / 16) {  // chunk et: positions p0, p0+1, ... (a prefill chunk) -> RoPE recurrence
          const int c0 = et * 16, n = min(16, tvalid - c0);
          int ok = 1;
          for (int j = 1; j < n; ++j) ok &= s_pos[c0 + j] == s_pos[c0] + j;
          s_consec[et] = ok;
        }
        named_bar_sync(2, kEpiThreads);
      }
      if (lane == 0) {
        if (ring)
          mbar_wait(&tfull[seg & 1], (seg >> 1) & 1);
        else
          mbar_wait(&tfull[buf], use & 1);
      }
      __syncwarp();
      tc_fence_after();
      if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg < 64) (DBG ? ep.trace : nullptr)[tb * 1024 + 512 + seg] = globaltimer_ns();
      const uint32_t trow = tmem + ((quarter * 32u) << 16);
      // TMEM drain with TWO of this warp's chunks in flight (one tcgen05.wait::ld per pair of
      // chunks): for epilogues whose per-chunk work is shorter than a TMEM load round trip
      // (partials, residual adds, plain stores), the drain would otherwise be latency-bound
      auto drain2 = [&](auto&& body) {
        if (eh >= nchunks) {
          release_tmem();
          return;
        }
        uint32_t ra[16], rb[16];
        const bool hb = eh + NEH < nchunks;
        tmem_ld_32x32b_x16(trow + tcol(eh), ra);
        if (hb) tmem_ld_32x32b_x16(trow + tcol(eh + NEH), rb);
        tmem_ld_wait_regs(ra);
        regs_fence(rb);
        after_load(eh);
        if (hb) after_load(eh + NEH);
        for (int ch = eh; ch < nchunks; ch += 2 * NEH) {
          uint32_t na[16], nb[16];
          const int c2 = ch + 2 * NEH, c3 = ch + 3 * NEH;
          const bool m2 = c2 < nchunks, m3 = c3 < nchunks;
          if (m2) tmem_ld_32x32b_x16(trow + tcol(c2), na);
          if (m3) tmem_ld_32x32b_x16(trow + tcol(c3), nb);
          body(ch, ra);
          if (ch + NEH < nchunks) body(ch + NEH, rb);
          if (m2) {
            tmem_ld_wait_regs(na);
            regs_fence(nb);
            after_load(c2);
            if (m3) after_load(c3);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              ra[j] = na[j];
              rb[j] = nb[j];
            }
          }
        }
      };
      if (direct) {
        // TMEM drain, one chunk in flight (load, wait, emit): measured faster than keeping the next
        // chunk's load in flight across the emit, for every epilogue mode (tools/tmem_drain.cu;
        // [13B-1] QKV 66.2 -> 64.8 us, gate||up 92.3 -> 89.8, O 30.8 -> 30.2; step 19.05 -> 18.85 ms,
        // interleaved A/B, profiles/r02_ab_drain.txt)
        if (c_lo + eh >= c_hi) {
          release_tmem();
        } else {
          for (int ch = c_lo + eh; ch < c_hi; ch += NEH) {
            uint32_t raw[16];
            tmem_ld_32x32b_x16(trow + tcol(ch), raw);
            tmem_ld_wait_regs(raw);
            after_load(ch);
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]);
            if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg == 0 && ch < 64)
              (DBG ? ep.trace : nullptr)[tb * 1024 + 800 + ch] = globaltimer_ns();
            if (!(DBG && (ep.dbg & 4)))
              epi_emit<MODE, DBG>(p.M, p.bn, ep, v, quarter, lane, mt, nt, ch * 16, tvalid, sbuf, s_pos, s_slot, s_consec, ql,
                       (DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg == 0 && ch < 64 ? (DBG ? ep.trace : nullptr) + tb * 1024 + 864 + ch : nullptr);
            if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg == 0 && ch < 64)
              (DBG ? ep.trace : nullptr)[tb * 1024 + 640 + ch] = globaltimer_ns();
          }
        }
      } else {
        // stream-K partial: slot = position of this pair among the tile's contributors; the last to
        // arrive sums the slots in slot order (deterministic) and runs the fused epilogue
        const int c_first = cta_of(static_cast<long long>(tile) * p.KB, p);
        const int c_last = cta_of(static_cast<long long>(tile) * p.KB + p.KB - 1, p);
        const int nslot = c_last - c_first + 1;
        const int slot = pair - c_first;
        const size_t tile128 = static_cast<size_t>(mt) * p.n_tiles + nt;
        // partial layout [chunk][lane quarter][token quad j][lane][4 tokens] (fp32): a thread keeps its
        // row's 16 tokens as four float4, and each warp-wide 16-B vector access is 512 contiguous bytes
        const size_t qoff = static_cast<size_t>(quarter) * 512 + lane * 4;  // + (ch * 4 * 512) + j * 128
        float* wsp = p.red_partials ? ep.ws_red + tile128 * tile_elems + qoff
                                    : ep.ws + (tile128 * p.max_slots + slot) * tile_elems + qoff;
        // TMEM is released right after the last load (drain2)
        drain2([&](int ch, uint32_t (&raw)[16]) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 x = make_float4(__uint_as_float(raw[4 * j]), __uint_as_float(raw[4 * j + 1]),
                                         __uint_as_float(raw[4 * j + 2]), __uint_as_float(raw[4 * j + 3]));
            if (p.red_partials)
              red_add_v4(wsp + ch * 2048 + j * 128, x);
            else
              __stcg(reinterpret_cast<float4*>(wsp + ch * 2048 + j * 128), x);
          }
        });
        if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg < 32) (DBG ? ep.trace : nullptr)[tb * 1024 + 704 + seg] = globaltimer_ns();
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg < 32) (DBG ? ep.trace : nullptr)[tb * 1024 + 736 + seg] = globaltimer_ns();
        if (et == 0) {
          int* ctr = ep.counters + tile128;
          const int old = atomicAdd(ctr, 1);
          s_last = (old == nslot - 1);
          if (s_last) *ctr = 0;  // re-arm for the next launch
        }
        named_bar_sync(1, kEpiThreads);
        if (s_last && eh < nchunks) {
          __threadfence();
          float* rowbase = p.red_partials ? ep.ws_red + tile128 * tile_elems + qoff
                                          : ep.ws + tile128 * p.max_slots * tile_elems + qoff;
          const int nsum = p.red_partials ? 1 : nslot;  // red.add already summed every contributor
          // slots summed in slot order (deterministic); slot 0 of the next chunk is in flight while
          // this chunk is summed and emitted (A/B register buffers, no copies)
          auto load1 = [&](int ch, float4 (&buf)[4]) {
#pragma unroll
            for (int j = 0; j < 4; ++j) buf[j] = __ldcg(reinterpret_cast<const float4*>(rowbase + ch * 2048 + j * 128));
          };
          auto sum_emit = [&](int ch, const float4 (&buf)[4]) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v[4 * j + 0] = buf[j].x;
              v[4 * j + 1] = buf[j].y;
              v[4 * j + 2] = buf[j].z;
              v[4 * j + 3] = buf[j].w;
            }
            for (int q = 1; q < nsum; ++q) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 x = __ldcg(reinterpret_cast<const float4*>(rowbase + q * tile_elems + ch * 2048 + j * 128));
                v[4 * j + 0] += x.x;
                v[4 * j + 1] += x.y;
                v[4 * j + 2] += x.z;
                v[4 * j + 3] += x.w;
              }
            }
            epi_emit<MODE, DBG>(p.M, p.bn, ep, v, quarter, lane, mt, nt, ch * 16, tvalid, sbuf, s_pos, s_slot, s_consec, ql);
          };
          float4 A[4], B[4];
          load1(eh, A);
          for (int ch = eh; ch < nchunks; ch += 2 * NEH) {
            if (ch + NEH < nchunks) load1(ch + NEH, B);
            sum_emit(ch, A);
            if (ch + NEH < nchunks) {
              if (ch + 2 * NEH < nchunks) load1(ch + 2 * NEH, A);
              sum_emit(ch + NEH, B);
            }
          }
          if (p.red_partials) {  // re-zero this thread's part of the slot for the next launch
            for (int ch = eh; ch < nchunks; ch += NEH)
#pragma unroll
              for (int j = 0; j < 4; ++j)
                __stcg(reinterpret_cast<float4*>(rowbase + ch * 2048 + j * 128), make_float4(0.f, 0.f, 0.f, 0.f));
          }
        }
      }
      if ((DBG ? ep.trace : nullptr) && tb < 2 && et == 0 && seg < 64) (DBG ? ep.trace : nullptr)[tb * 1024 + 576 + seg] = globaltimer_ns();
      ++seg;
    }
  }

  if (MODE == EPI_ADD_F32 && ep.pnorm_out) {
    // RMSNorm of the updated residual stream (the next GEMM's input) by this grid: every CTA's
    // residual adds land (fence + grid barrier on the monotonic counter; all CTAs of the persistent
    // grid are resident), then the CTAs normalise rows blockIdx.x, blockIdx.x + grid, ...  Replaces
    // the rmsnorm launch and its grid-completion gap.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(ep.norm_ctr, 1u);
      xflag_wait(ep.norm_ctr, ep.norm_target);
    }
    __syncthreads();
    norm_rows<64 + 128 * NEH>(static_cast<const float*>(ep.out), static_cast<const __nv_bfloat16*>(ep.pnorm_g),
                              static_cast<__nv_bfloat16*>(ep.pnorm_out), ep.norm_T, ep.norm_H, ep.norm_eps, stage_buf);
  }
  if (ep.done_ctr) __threadfence();  // this thread's stores / red.adds before the CTA's count
  tc_fence_before();
  __syncthreads();
  if (ep.done_ctr && threadIdx.x == 0) atomicAdd(ep.done_ctr, 1u);
  if (ep.span_end && threadIdx.x == 0) atomicMax(ep.span_end, globaltimer_ns());
  if ((DBG ? ep.trace : nullptr) && threadIdx.x == 0) {
    (DBG ? ep.trace : nullptr)[2048 + blockIdx.x] = globaltimer_ns();  // per-CTA end (debug)
    if (blockIdx.x == 0) (DBG ? ep.trace : nullptr)[2047] = 1;
  }
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, p.tmem_cols);
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

// epilogue warps per TMEM lane quarter: 2 (3 and 4 were measured: no faster / slower with spills)
constexpr int kNEH = 2;
size_t extra_smem(int bn) {
  return 4 * kNEH * kStageFloats * 4 + 32 * 4 + 2 * static_cast<size_t>(bn) * 4 + 3 * 8 * 8 + 64 + 64;
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

GemmPlan plan_gemm(int M, int N, int K, int num_sms, size_t ws_cap_floats, int force_pairs, bool atomic_epilogue,
                   bool deterministic) {
  if (deterministic) atomic_epilogue = false;  // residual adds reduce through slots as well
  GemmPlan pl;
  pl.atomic = atomic_epilogue ? 1 : 0;
  pl.M = M;
  pl.N = N;
  pl.K = K;
  const int KB = K / kBK;
  const TokenTiling tt = gemm_token_tiling(N);  // shared with the scheduler's chunk advisor
  pl.n_tiles = tt.n_tiles;
  pl.n_mma = tt.n_mma;
  pl.bn = tt.bn;
  {
    // Few weight-row tiles (a TP rank's small M) or, for residual adds, a short K: two token
    // tiles spread the exposed epilogue (and halve the split-K red.add volume) over twice the CTA
    // pairs.  Measured (tools/shard_step.py, profiles/r02_shard_step.txt): LLaMA-2-70B TP-8 rank
    // QKV 37.9 -> 26.4 us, O 13.6 -> 11.7, gate||up 51.8 -> 44.6 (per layer 172.7 -> 158.8 us);
    // but the 13B TP-1 O / down (K = 5120 / 13824) got slower (23.8 -> 30.8, 46 -> 72 us), hence
    // the K bound for residual adds.  SARATHI_GEMM_NT_SMALLM=n overrides the split (0 = off).
    static const int nt_small = getenv("SARATHI_GEMM_NT_SMALLM") ? atoi(getenv("SARATHI_GEMM_NT_SMALLM")) : 2;
    const int pm = (M + 2 * kBM - 1) / (2 * kBM);
    // (GPT-3 TP-8 rank, K = 12288: QKV 52.6 -> 55.4, gate 53.6 -> 65.9 us with the split, so long
    // K keeps the full token tile: the mainloop dominates and narrow UMMAs cost more than the
    // epilogue saves)
    // (residual adds: only up to 16 k-blocks; the GPT-3 TP-8 rank's O, K = 1536, measured 23.1 us
    // split vs 19.4 unsplit, tools/shard_sweep.sh, profiles/r02_shard_sweep.txt)
    const bool small = atomic_epilogue ? KB <= 16 : (2 * pm * tt.n_tiles < num_sms / 2 && KB <= 128);
    if (nt_small > tt.n_tiles && force_pairs == 0 && small) {
      pl.n_tiles = nt_small;
      const int per = (N + nt_small - 1) / nt_small;
      pl.n_mma = per <= 256 ? 1 : 2;
      pl.bn = per <= 256 ? std::max(16, (per + 15) / 16 * 16) : (per + 31) / 32 * 32;
    }
  }
  pl.box_rows = pl.bn / pl.n_mma / 2;  // each CTA of the pair holds half of every UMMA's tokens
  pl.n0 = pl.n1 = pl.bn / pl.n_mma;
  pl.box_rows2 = pl.box_rows;
  pl.pm_tiles = (M + 2 * kBM - 1) / (2 * kBM);
  pl.m_tiles = 2 * pl.pm_tiles;
  const int tiles = pl.pm_tiles * pl.n_tiles;
  pl.tiles = tiles;
  const int P = std::max(1, num_sms / 2);
  // Work split (in k-block units; a split tile costs a partial write + a reduction, ~KB/2 units
  // when it is exposed at the kernel end):
  //  * residual-add epilogues reduce with red.add (no reduction pass): pure stream-K over all pairs;
  //  * tiles <= P: one whole tile per pair (data-parallel) unless stream-K saves > KB/2 units;
  //  * tiles > P: the tiles % P remainder stream-K first (reductions overlap the rest), then
  //    tiles / P whole tiles per pair.
  int pairs, sk_tiles, dp_per, dp_extra = 0;
  if (force_pairs > 0) {
    pairs = static_cast<int>(std::min<long long>(static_cast<long long>(tiles) * KB, force_pairs));
    sk_tiles = tiles;
    dp_per = 0;
  } else if (atomic_epilogue) {
    // residual adds reduce with red.add: split-K.  With tiles <= pairs, split every tile the same
    // number of ways (pairs = tiles * floor(P / tiles)) so each pair's k-range lies inside ONE tile:
    // one red.add epilogue per pair instead of two for ranges straddling a tile boundary
    pairs = static_cast<int>(std::min<long long>(P, std::max<long long>(1, static_cast<long long>(tiles) * KB / 4)));
    // (only for wide token tiles: with small bn the red.add epilogue is cheap and every pair counts)
    if (tiles <= P && pl.bn >= 128 && !getenv("SARATHI_GEMM_SK_ANY"))
      pairs = tiles * std::max(1, std::min(P / tiles, KB / 4));
    sk_tiles = tiles;
    dp_per = 0;
  } else if (tiles <= P) {
    const int sk_pairs = static_cast<int>(std::min<long long>(P, std::max<long long>(1, static_cast<long long>(tiles) * KB / 4)));
    // cost model in k-block units: a split tile adds a partial write + reduction ~ sk_cost * KB
    static const double sk_cost = getenv("SARATHI_GEMM_SK_COST") ? atof(getenv("SARATHI_GEMM_SK_COST")) : 0.5;
    const double sk_units = std::ceil(static_cast<double>(tiles) * KB / sk_pairs) + sk_cost * KB;
    if (KB <= sk_units) {
      pairs = tiles;
      sk_tiles = 0;
      dp_per = 1;
    } else {
      pairs = sk_pairs;
      sk_tiles = tiles;
      dp_per = 0;
    }
  } else {
    pairs = P;
    dp_per = tiles / P;
    sk_tiles = tiles % P;
    // Token-half remainder: with two equal UMMAs per k-step (ring accumulator), the tiles % P
    // remainder tiles are split over their two token halves instead of over K, one half per pair
    // after its whole tiles: no partials, no reduction pass, and the first whole tile's epilogue
    // overlaps the half item's mainloop.  LLaMA-13B gate||up at T = 320 (108 tiles on 74 pairs):
    // the stream-K remainder's partial drain stalled the next segment and its last contributors'
    // reductions formed the kernel's tail (tools/experiments.sh layer).  SARATHI_GEMM_HALF=0 disables.
    static const bool half_on = !(getenv("SARATHI_GEMM_HALF") && atoi(getenv("SARATHI_GEMM_HALF")) == 0);
    const bool ring_shape = pl.n_tiles == 1 && pl.n_mma == 2 && 3 * (pl.bn / 2) <= 512 && N > pl.bn / 2;
    if (half_on && !atomic_epilogue && ring_shape && sk_tiles > 0 && 2 * sk_tiles <= P) {
      pl.half_items = 2 * sk_tiles;
      sk_tiles = 0;
    } else if (static_cast<long long>(sk_tiles) * KB < 4LL * P) {  // remainder too small to split: whole tiles
      dp_extra = sk_tiles;
      sk_tiles = 0;
    }
  }
  const long long units = static_cast<long long>(sk_tiles) * KB;
  auto slots_for = [&](int g) {
    if (units == 0) return 1;
    const long long pc = std::max<long long>(1, units / g);
    const int s = pc >= KB ? 2 : static_cast<int>((KB + pc - 1) / pc) + 1;
    return std::min(s, g);
  };
  int max_slots = slots_for(pairs);
  const size_t tile_elems = static_cast<size_t>(pl.bn) * kBM;
  const size_t tiles128 = static_cast<size_t>(pl.m_tiles) * pl.n_tiles;
  // more than 4 contributors per split tile (few row tiles, e.g. a TP-8 rank's QKV): accumulate the
  // partials by red.add into one zeroed fp32 slot per tile (the last contributor reads it once, runs
  // the epilogue and re-zeroes it) instead of shrinking the grid to <= 4 slots
  pl.red_partials = 0;
  if (!deterministic && !atomic_epilogue && dp_per == 0 && max_slots > 4 && tiles128 * tile_elems <= ws_cap_floats / 2) {
    pl.red_partials = 1;
    max_slots = 1;
  }
  while (!atomic_epilogue && !pl.red_partials && dp_per == 0 && pairs > 1 && max_slots > 4) {
    --pairs;
    max_slots = slots_for(pairs);
  }
  while (!atomic_epilogue && !pl.red_partials && dp_per == 0 && pairs > 1 &&
         tiles128 * max_slots * tile_elems > ws_cap_floats / 2) {
    pairs = std::max(1, pairs / 2);
    max_slots = slots_for(pairs);
  }
  pl.ctas = pairs;
  pl.sk_tiles = sk_tiles;
  pl.dp_per_pair = dp_per;
  pl.dp_extra = dp_extra;
  pl.units = units;
  pl.max_slots = max_slots;
  pl.splits = static_cast<int>((units + pairs - 1) / pairs) + dp_per * KB;  // units per pair (informational)
  pl.kb_per_split = pl.splits;
  pl.ws_floats = units > 0 && !atomic_epilogue && !pl.red_partials ? tiles128 * max_slots * tile_elems : 0;
  pl.nbuf = pl.bn <= 256 ? 2 : 1;
  // Uneven split for 256 < T <= 512 when every pair runs ONE segment (nothing to overlap a second
  // accumulator with): UMMA 0 takes 256 tokens, UMMA 1 the 16-multiple tail, so T = 257 costs
  // 256 + 16 token columns instead of 2 x 144 (the B200 form of the paper's tile quantization,
  // P:L457-463).  SARATHI_GEMM_UNEVEN=0 keeps the equal halves.
  {
    static const bool uneven_on = !(getenv("SARATHI_GEMM_UNEVEN") && atoi(getenv("SARATHI_GEMM_UNEVEN")) == 0);
    int max_segs = 0;
    for (int c = 0; c < pl.ctas; ++c) {
      const long long u0 = static_cast<long long>(c) * pl.units / pl.ctas, u1 = static_cast<long long>(c + 1) * pl.units / pl.ctas;
      const int sk = u1 > u0 ? static_cast<int>((u1 - 1) / KB - u0 / KB + 1) : 0;
      max_segs = std::max(max_segs, sk + pl.dp_per_pair + (c < pl.dp_extra ? 1 : 0) + (c < pl.half_items ? 1 : 0));
    }
    const int per = (N + pl.n_tiles - 1) / pl.n_tiles;
    if (uneven_on && pl.n_mma == 2 && pl.n_tiles == 1 && max_segs <= 1 && per > 256 && per <= 512) {
      pl.n0 = 256;
      pl.n1 = std::max(16, (per - 256 + 15) / 16 * 16);
      pl.bn = pl.n0 + pl.n1;
      pl.box_rows = 128;
      pl.box_rows2 = pl.n1 / 2;
      pl.nbuf = 1;
    }
  }
  const size_t stage = kABytes + static_cast<size_t>(pl.bn / 2) * kBK * 2;
  const size_t budget = 226 * 1024 - 1024 - extra_smem(pl.bn);
  pl.stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(8, budget / stage)));
  pl.smem = pl.stages * stage + extra_smem(pl.bn) + 1024;
  return pl;
}

bool make_tmap_f32_red(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 4};
  cuuint32_t box[2] = {32, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_weight(CUtensorMap* map, const void* w, int M, int K) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) return false;
  const uint64_t rows = static_cast<uint64_t>((M + kBM - 1) / kBM) * (K / kBK) * kWRowsPerTile;
  cuuint64_t dims[2] = {256, rows};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {256, kWRowsPerTile};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void dump_gemm_trace(const unsigned long long* trace_dev, const GemmPlan& pl) {
  static unsigned long long h[4096];
  cudaMemcpy(h, trace_dev, sizeof(h), cudaMemcpyDeviceToHost);
  const unsigned long long t0 = h[0];
  fprintf(stderr, "gemm trace M=%d N=%d K=%d pairs=%d stages=%d units/pair~%lld\n", pl.M, pl.N, pl.K, pl.ctas, pl.stages,
          pl.units / std::max(1, pl.ctas));
  for (int i = 0; i < 256 && h[i]; ++i)
    fprintf(stderr, "u%3d issue0 %8.3f issue1 %8.3f mma %8.3f us\n", i, (h[i] - t0) * 1e-3,
            h[1024 + i] ? (h[1024 + i] - t0) * 1e-3 : -1.0, h[256 + i] ? (h[256 + i] - t0) * 1e-3 : -1.0);
  {
    int n = 0;
    std::vector<double> ends;
    for (int b = 0; b < 2 * pl.ctas && 2048 + b < 4096; ++b)
      if (h[2048 + b]) {
        ends.push_back((h[2048 + b] - t0) * 1e-3);
        ++n;
      }
    std::sort(ends.begin(), ends.end());
    if (n) fprintf(stderr, "CTA end times (us): min %.2f p25 %.2f p50 %.2f p75 %.2f max %.2f (n=%d)\n", ends[0],
                   ends[n / 4], ends[n / 2], ends[3 * n / 4], ends[n - 1], n);
    if (getenv("SARATHI_TRACE_ALL")) {
      for (int b = 0; b < 2 * pl.ctas; b += 2)
        fprintf(stderr, "pair %d end %.2f\n", b / 2, h[2048 + b] ? (h[2048 + b] - t0) * 1e-3 : -1.0);
    }
  }
  for (int ch = 0; ch < 64; ++ch)
    if (h[640 + ch]) fprintf(stderr, "seg0 chunk %d loaded %8.3f  regs-done %8.3f  emitted %8.3f us\n", ch,
            h[800 + ch] ? (h[800 + ch] - t0) * 1e-3 : -1.0, h[864 + ch] ? (h[864 + ch] - t0) * 1e-3 : -1.0,
            (h[640 + ch] - t0) * 1e-3);
  for (int sgm = 0; sgm < 64 && h[512 + sgm]; ++sgm)
    fprintf(stderr, "seg %d epilogue wake %8.3f us  done %8.3f us  (partial stored %8.3f, fenced %8.3f)\n", sgm,
            (h[512 + sgm] - t0) * 1e-3, h[576 + sgm] ? (h[576 + sgm] - t0) * 1e-3 : -1.0,
            sgm < 32 && h[704 + sgm] ? (h[704 + sgm] - t0) * 1e-3 : -1.0,
            sgm < 32 && h[736 + sgm] ? (h[736 + sgm] - t0) * 1e-3 : -1.0);
}

cudaError_t launch_gemm(const CUtensorMap& mapW, const CUtensorMap& mapX, const CUtensorMap& mapX2, const GemmPlan& pl,
                        const EpiParams& ep, cudaStream_t stream) {
  // one kernel per (epilogue mode, debug) so the epilogue has no runtime mode switch (smaller code,
  // fewer branches); debug/trace instrumentation only in the DBG instantiations
  using KFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const KParams, const EpiParams);
  static const KFn table[2][6] = {
      {gemm_bf16_pair<kNEH, 0, false>, gemm_bf16_pair<kNEH, 1, false>, gemm_bf16_pair<kNEH, 2, false>,
       gemm_bf16_pair<kNEH, 3, false>, gemm_bf16_pair<kNEH, 4, false>, gemm_bf16_pair<kNEH, 5, false>},
      {gemm_bf16_pair<kNEH, 0, true>, gemm_bf16_pair<kNEH, 1, true>, gemm_bf16_pair<kNEH, 2, true>,
       gemm_bf16_pair<kNEH, 3, true>, gemm_bf16_pair<kNEH, 4, true>, gemm_bf16_pair<kNEH, 5, true>}};
  static bool configured = false;
  if (!configured) {
    for (auto& row : table)
      for (KFn fn : row) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (e != cudaSuccess) return e;
        prefer_max_smem(fn);
      }
    configured = true;
  }
  if (ep.mode < 0 || ep.mode > 5) return cudaErrorInvalidValue;
  const KFn fn = table[(ep.dbg || ep.trace) ? 1 : 0][ep.mode];
  static const bool kbasm_on = !(getenv("SARATHI_GEMM_KBASM") && atoi(getenv("SARATHI_GEMM_KBASM")) == 0);
  EpiParams epk = ep;
  epk.kbasm = kbasm_on ? 1 : 0;
  static const bool relaxed_on = !(getenv("SARATHI_GEMM_RELAXED") && atoi(getenv("SARATHI_GEMM_RELAXED")) == 0);
  epk.relaxed_rel = relaxed_on ? 1 : 0;
  KParams kp;
  kp.M = pl.M;
  kp.N = pl.N;
  kp.KB = pl.K / kBK;
  kp.bn = pl.bn;
  kp.n_mma = pl.n_mma;
  kp.pm_tiles = pl.pm_tiles;
  kp.n_tiles = pl.n_tiles;
  kp.units = pl.units;
  kp.ctas = pl.ctas;
  kp.sk_tiles = pl.sk_tiles;
  kp.dp_per_pair = pl.dp_per_pair;
  kp.dp_extra = pl.dp_extra;
  kp.half_items = pl.half_items;
  kp.tiles = pl.tiles;
  kp.stages = pl.stages;
  kp.nbuf = pl.nbuf;
  kp.n0 = pl.n0;
  kp.n1 = pl.n1;
  kp.max_slots = pl.max_slots;
  kp.red_partials = pl.red_partials;
  kp.atomic = pl.atomic;
  kp.tmem_cols = (pl.nbuf == 2 || (pl.n_mma == 2 && 3 * (pl.bn / 2) <= 512)) ? 512 : pow2_cols(pl.bn);
  {
    // A from TMEM for two-UMMA k-steps (T > 256) whose accumulators leave columns [kTsCol, 512)
    // free (ring of 3 x <= 160, or one accumulator of <= 480 tokens): tcgen05.cp stages each k16
    // slice of the weight tile once and both UMMAs read it from TMEM, instead of each UMMA
    // re-reading it from shared memory (the second UMMA of a k-step cost ~0.13 us per k-block
    // whatever its width: shared-memory operand bandwidth).  Measured at [13B-1]: per-k-block
    // 0.48 -> 0.448 us (N = 320, tools/experiments.sh ts), layer GEMMs 240 -> 226 us, step 19.00 ->
    // 18.51 ms (interleaved A/B, profiles/r02_ab_ts.txt).  SARATHI_GEMM_TS=0 disables.
    static const bool ts_on = !(getenv("SARATHI_GEMM_TS") && atoi(getenv("SARATHI_GEMM_TS")) == 0);
    const bool ring = pl.n_mma == 2 && pl.n0 == pl.n1 && 3 * pl.n0 <= 512;
    const int used = pl.n_mma != 2 ? 512 : ring ? 3 * pl.n0 : pl.bn;
    kp.ts = ts_on && pl.n_mma == 2 && used <= kTsCol;
    if (kp.ts) kp.tmem_cols = 512;
  }
  kp.ring_bytes = static_cast<uint32_t>(pl.stages * (kABytes + static_cast<size_t>(pl.bn / 2) * kBK * 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pl.ctas);
  cfg.blockDim = dim3(threads_of<kNEH>());
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see the producer)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fn, mapW, mapX, mapX2, kp, epk);
}

}  // namespace sarathi

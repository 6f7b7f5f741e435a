// Layer chain: the four linears of one transformer layer's GEMM phase as ONE persistent tcgen05
// launch — O-proj + residual ("postproj"), FFN1 (ffn_ln1 + SiLU*up / GELU), FFN2
// + residual (ffn_ln2), then the NEXT layer's QKV + RoPE + KV append (preproj) — over the same
// hybrid-batch token matrix (decode-maximal batching fuses every linear over all p + d tokens,
// PAPER.md L403-407 §4.3).
//
// Why one launch (B200 design): at T ≈ 320 tokens each linear is a few tens of
// microseconds of MMA work on 74 CTA pairs, and a per-GEMM launch pays pipeline fill, an exposed
// last-tile epilogue, tile quantization (QKV: 60 pair tiles on 74 pairs, gate||up 108 on 74) and a
// kernel boundary + RMSNorm launch between every two linears.  Here every CTA pair walks a host-
// planned list of segments (job, 256-row pair tile, k-block range; host_sched.cpp schedule_chain),
// and job j+1 reads job j's output tile by tile through release/acquire flags:
//   * the TMA producer, before loading X k-block kb of job j+1, waits for the 128-row output tile
//     of job j that holds those 64 columns (flag >= epoch), then orders the async proxy after it;
//   * a residual-add job (O, FFN2) red.adds its split-K partial into the fp32 residual h; the last
//     contributor of a 128-column tile (arrival counter) finalises it: X' = bf16(g * h) for the
//     next job and the per-token sum of squares of those 128 columns (the RMSNorm statistics,
//     summed over tiles in tile order, so the scale is deterministic);
//   * the consuming job's epilogue multiplies token t's accumulator by rsqrt(sum / H + eps) before
//     its activation: RMSNorm(h) W^T = rs_t * (g∘h) W^T (reading O-8; no RMSNorm kernel).
// Warp roles, TMEM ring / double buffer and the epilogue bodies are the single-GEMM kernel's
// (gemm.cu, gemm_epi.cuh).  All CTAs are co-resident (grid = one CTA per SM), waits only point to
// earlier jobs, and every pair runs its segments in job order, so the dependency graph is acyclic;
// a wait that exceeds 4 s traps (a lost dependency fails loudly instead of hanging the GPU).
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "host_sched.hpp"

#include <algorithm>

namespace sarathi {

namespace {

constexpr int kNEHc = 2;  // epilogue warps per TMEM lane quarter (as gemm.cu)

SARATHI_DEVICE unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SARATHI_DEVICE unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SARATHI_DEVICE void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
SARATHI_DEVICE void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy global writes <-> async-proxy (TMA) reads of the same data
SARATHI_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Spin with relaxed loads (an acquire load per iteration also invalidates L1: CCTL.IVALL), then one
// acquire fence once the flag is seen.
SARATHI_DEVICE void wait_flag(const unsigned* f, unsigned epoch) {
  if (static_cast<int>(ld_acquire_gpu(f) - epoch) >= 0) return;
  const unsigned long long t0 = globaltimer_ns();
  while (static_cast<int>(ld_relaxed_gpu(f) - epoch) < 0) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
  fence_acq_rel_gpu();
}

// Bulk reduce-add of a warp's 16-token x 32-column fp32 block (token-major in shared memory) into
// global memory through the TMA engine (one 2 KB request instead of 128 vector red.adds).
SARATHI_DEVICE void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
SARATHI_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SARATHI_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SARATHI_DEVICE void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
SARATHI_DEVICE void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Seg {
  int job, pt, kb0, kb1;
};
SARATHI_DEVICE Seg load_seg(const int* segs, int i) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(segs) + i);
  return Seg{v.x, v.y, v.z, v.w};
}

size_t chain_extra_smem(int bn) {
  // 2 sets of transpose buffers + s_pos/s_slot (2 bn ints) + s_consec[32] + s_rs[bn] + barriers + holder
  return 2 * 4 * kNEHc * kStageFloats * 4 + 32 * 4 + 3 * static_cast<size_t>(bn) * 4 + 3 * 8 * 8 + 16 * 8 + 64 + 64;
}

template <int FFN>
__global__ void __launch_bounds__(threads_of<kNEHc>(), 1)
    gemm_chain_pair(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainLaunch p) {
  constexpr int NEH = kNEHc;
  constexpr int kEpiThreads = 128 * NEH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t b_bytes = static_cast<uint32_t>(p.bn / 2) * kBK * 2;  // this CTA's half of the tokens
  const uint32_t stage_bytes = kABytes + b_bytes;
  float* stage_buf = reinterpret_cast<float*>(smem + p.ring_bytes);       // [2][8 warps][16 x 32]
  int* s_pos = reinterpret_cast<int*>(stage_buf + 2 * 4 * NEH * kStageFloats);  // [bn]
  int* s_slot = s_pos + p.bn;                                               // [bn]
  int* s_consec = s_slot + p.bn;                                            // [32]
  float* s_rs = reinterpret_cast<float*>(s_consec + 32);                    // [bn] per-token RMSNorm scale
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_rs + p.bn);
  uint64_t* full = bars;
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;  // [2]
  uint64_t* tempty = tfull + 2;        // [3]
  uint64_t* sbar = tempty + 3;         // [8 epilogue warps][2] split-tile scratch loads
  uint32_t* holder = reinterpret_cast<uint32_t*>(sbar + 8 * NEH);
  __shared__ int s_last;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  griddep_launch_dependents();
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[static_cast<size_t>(gridDim.x / 2) * kChainTraceSegs * 8] = globaltimer_ns();
  const int pair = blockIdx.x >> 1;
  const int seg_begin = __ldg(p.seg_off + pair), seg_end = __ldg(p.seg_off + pair + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&tfull[b], 1);
    for (int b = 0; b < 3; ++b) mbar_init(&tempty[b], 8 * NEH);
    for (int b = 0; b < 8 * NEH; ++b) mbar_init(&sbar[b], 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    for (int j = 0; j < p.njobs; ++j) {
      tma_prefetch_desc(&maps.w[j]);
      tma_prefetch_desc(&maps.x[j]);
    }
  }
  if (warp == 1) tmem_alloc_pair(holder, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const int ni = p.bn / p.n_mma;
  const bool ring = p.n_mma == 2 && 3 * ni <= 512;
  if (warp != 0) griddep_wait();
  // device span from the end of the grid dependency (the predecessor's completion), not residency
  if (p.span_start && threadIdx.x == 64) atomicMin(p.span_start, globaltimer_ns());
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 64) p.trace[static_cast<size_t>(gridDim.x / 2) * kChainTraceSegs * 8 + 1] = globaltimer_ns();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    const uint32_t tx = 2 * stage_bytes;
    int s = 0;
    uint32_t ph = 0;
    int i = 0, npre = 0;
    if (seg_begin < seg_end) {  // PDL: the first segment's W tiles before the grid dependency
      const Seg sg = load_seg(p.segs, seg_begin);
      const int KB = p.job[sg.job].KB;
      npre = min(p.stages, sg.kb1 - sg.kb0);
      const int wrow0 = ((sg.pt * 2 + static_cast<int>(rank)) * KB + sg.kb0) * kWRowsPerTile;
      for (int j = 0; j < npre; ++j) {
        if (rank == 0) mbar_arrive_expect_tx_warp(&full[j], tx);
        tma_load_2d_pair_warp(smem + static_cast<size_t>(j) * stage_bytes, &maps.w[sg.job], &full[j], 0,
                              wrow0 + j * kWRowsPerTile, pol_w);
      }
    }
    griddep_wait();
    for (int si = seg_begin; si < seg_end; ++si) {
      const Seg sg = load_seg(p.segs, si);
      const ChainJobDev& J = p.job[sg.job];
      const CUtensorMap* mw = &maps.w[sg.job];
      const CUtensorMap* mx = &maps.x[sg.job];
      int wrow = ((sg.pt * 2 + static_cast<int>(rank)) * J.KB + sg.kb0) * kWRowsPerTile;
      int have = -1;  // dependency tile already acquired in this segment
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++i) {
        uint8_t* a = smem + static_cast<size_t>(s) * stage_bytes;
        uint8_t* b = a + kABytes;
        if (i >= npre) {
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx_warp(&full[s], tx);
          tma_load_2d_pair_warp(a, mw, &full[s], 0, wrow, pol_w);  // weights: no dependency
        }
        if (J.dep_flag) {
          const int need = kb >> J.dep_shift;
          if (need > have) {
            // one warp-wide relaxed scan of the next 32 dependency tiles (instead of an acquire per
            // tile), one acquire fence for all of them, one proxy fence before the TMA reads
            const unsigned long long tw = p.trace ? globaltimer_ns() : 0;
            const int last = (sg.kb1 - 1) >> J.dep_shift;
            while (true) {
              const int q = need + static_cast<int>(lane);
              bool ok = true;
              if (q <= last) ok = static_cast<int>(ld_relaxed_gpu(J.dep_flag + q) - p.epoch) >= 0;
              const unsigned bad = __ballot_sync(0xffffffffu, !ok);
              const int nready = bad ? __ffs(bad) - 1 : 32;
              if (nready > 0) {
                have = need + nready - 1;
                break;
              }
              wait_flag(J.dep_flag + need, p.epoch);  // the first one is not ready: block on it
            }
            fence_acq_rel_gpu();
            fence_proxy_async_global();
            if (p.trace && rank == 0 && lane == 0 && si - seg_begin < kChainTraceSegs)
              p.trace[(static_cast<size_t>(pair) * kChainTraceSegs + (si - seg_begin)) * 8 + 5] += globaltimer_ns() - tw;
          }
        }
        tma_load_2d_pair_warp(b, mx, &full[s], kb * kBK, static_cast<int>(rank) * (ni / 2), pol_x);
        if (p.n_mma == 2)
          tma_load_2d_pair_warp(b + (ni / 2) * kBK * 2, mx, &full[s], kb * kBK, ni + static_cast<int>(rank) * (ni / 2),
                                pol_x);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
        wrow += kWRowsPerTile;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const uint32_t idesc = make_idesc_bf16_f32(2 * kBM, ni);
      int seg = 0, s = 0;
      uint32_t ph = 0;
      int uses[3] = {0, 0, 0};
      for (int si = seg_begin; si < seg_end; ++si, ++seg) {
        const Seg sg = load_seg(p.segs, si);
        const int buf = seg % p.nbuf;
        const uint32_t use = seg / p.nbuf;
        uint32_t d0, d1;
        int tb_idx;
        if (ring) {
          const int sa = (2 * seg) % 3, sb = (2 * seg + 1) % 3;
          for (int k : {sa, sb}) {
            if (uses[k]) mbar_wait_cluster(&tempty[k], (uses[k] - 1) & 1);
            ++uses[k];
          }
          d0 = tmem + sa * ni;
          d1 = tmem + sb * ni;
          tb_idx = seg & 1;
        } else {
          mbar_wait_cluster(&tempty[buf], (use & 1) ^ 1);
          d0 = tmem + buf * 256;
          d1 = d0 + ni;
          tb_idx = buf;
        }
        tc_fence_after();
        unsigned long long* tr = (p.trace && seg < kChainTraceSegs && lane == 0)
                                     ? p.trace + (static_cast<size_t>(pair) * kChainTraceSegs + seg) * 8
                                     : nullptr;
        if (tr) tr[0] = globaltimer_ns();
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (tr && kb == sg.kb0) tr[1] = globaltimer_ns();
          const uint32_t a = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
          const uint32_t b = a + kABytes;
          if (p.kbasm) {  // the whole k-block from one asm block (gemm.cu: per-UMMA issue paced the mainloop)
            umma_kblock_ss_pair(d0, d1, make_desc_k_sw128(a), make_desc_k_sw128(b), make_desc_k_sw128(b + (ni / 2) * 128),
                                idesc, idesc, kb != sg.kb0 ? 1u : 0u, p.n_mma == 2 ? 1u : 0u);
          } else {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint32_t acc = (kb != sg.kb0 || k != 0) ? 1u : 0u;
              umma_f16_ss_pair_warp(d0, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + k * 32), idesc, acc);
              if (p.n_mma == 2)
                umma_f16_ss_pair_warp(d1, make_desc_k_sw128(a + k * 32), make_desc_k_sw128(b + (ni / 2) * 128 + k * 32),
                                      idesc, acc);
            }
          }
          umma_commit_pair_mc_warp(&empty[s], 0x3);
          if (kb == sg.kb1 - 1) umma_commit_pair_mc_warp(&tfull[tb_idx], 0x3);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        if (tr) {
          tr[2] = globaltimer_ns();
          tr[6] = (static_cast<unsigned long long>(sg.job) << 48) | (static_cast<unsigned long long>(sg.pt) << 32) |
                  (static_cast<unsigned long long>(sg.kb0) << 16) | static_cast<unsigned long long>(sg.kb1);
        }
      }
    }
  } else {
    // ---------------- Epilogue (warps 2..9 of both CTAs) ----------------
    const int et = threadIdx.x - 64;
    const int ew = static_cast<int>(warp) - 2;
    const int eh = ew >> 2;
    const uint32_t quarter = warp & 3;
    float* sbuf = stage_buf + ew * kStageFloats;
    float* sbuf2 = stage_buf + (4 * NEH + ew) * kStageFloats;  // second buffer (bulk reduce double buffering)
    int red_par = 0;
    uint32_t sph[2] = {0, 0};  // phases of this warp's two scratch-load barriers
    int rs_job = -1;           // job whose per-token RMSNorm scales s_rs holds
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    const int tvalid = p.N;
    const int nchunks = (tvalid + 15) / 16;
    int seg = 0;
    for (int si = seg_begin; si < seg_end; ++si, ++seg) {
      const Seg sg = load_seg(p.segs, si);
      const ChainJobDev& J = p.job[sg.job];
      const EpiParams& ep = J.ep;
      const int mode = ep.mode;
      const int mt = sg.pt * 2 + static_cast<int>(rank);
      const int buf = seg % p.nbuf;
      const uint32_t use = seg / p.nbuf;
      const bool scaled = J.ss_in != nullptr;
      QkvLane ql{};
      if (mode == EPI_QKV_ROPE) ql = qkv_lane(ep, mt, quarter, lane);
      const int nA = ring ? ni / 16 : (1 << 30);
      const int sA = (2 * seg) % 3, sB = (2 * seg + 1) % 3;
      auto tcol = [&](int ch) -> uint32_t {
        if (!ring) return static_cast<uint32_t>(buf * 256 + ch * 16);
        return static_cast<uint32_t>(ch < nA ? sA * ni + ch * 16 : sB * ni + (ch - nA) * 16);
      };
      auto arrive_slot = [&](int k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (p.relaxed)
            mbar_arrive_cluster_relaxed(tempty_leader + k * 8);
          else
            mbar_arrive_cluster(tempty_leader + k * 8);
        }
      };
      auto last_of = [&](int lim) {
        if (lim <= eh) return -1;
        return eh + ((lim - 1 - eh) / NEH) * NEH;
      };
      const int lastA = last_of(min(nA, nchunks)), lastAll = last_of(nchunks);
      auto release_tmem = [&]() {
        if (ring) {
          arrive_slot(sA);
          arrive_slot(sB);
        } else {
          arrive_slot(buf);
        }
      };
      auto after_load = [&](int c) {
        if (ring) {
          if (c == lastA) arrive_slot(sA);
          if (c == lastAll) arrive_slot(sB);
        } else if (c == lastAll) {
          arrive_slot(buf);
        }
      };
      // per-segment staging (overlaps this segment's mainloop)
      if (mode == EPI_QKV_ROPE) {
        named_bar_sync(2, kEpiThreads);
        for (int t = et; t < tvalid; t += kEpiThreads) {
          s_pos[t] = __ldg(ep.pos + t);
          const int sl = __ldg(ep.slot + t);
          s_slot[t] = (sl / ep.block_size) * ep.n_kv_local * ep.block_size + sl % ep.block_size;
        }
        named_bar_sync(2, kEpiThreads);
        if (et < nchunks) {
          const int c0 = et * 16, n = min(16, tvalid - c0);
          int ok = 1;
          for (int j = 1; j < n; ++j) ok &= s_pos[c0 + j] == s_pos[c0] + j;
          s_consec[et] = ok;
        }
      }
      const bool new_rs = scaled && rs_job != sg.job;  // once per job and CTA (consecutive segments share it)
      if (new_rs) {
        // the RMSNorm statistics of the input: every producer tile published (acquire), then the
        // per-token sum of squares over the tiles in tile order (8 independent loads in flight)
        rs_job = sg.job;
        if (ew == 0)
          for (int q = static_cast<int>(lane); q < J.ss_parts; q += 32) wait_flag(J.dep_flag + q, p.epoch);
        named_bar_sync(2, kEpiThreads);
        for (int t = et; t < tvalid; t += kEpiThreads) {
          const float* src = J.ss_in + t;
          float acc = 0.f;
          int q = 0;
          for (; q + 8 <= J.ss_parts; q += 8) {
            float x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = __ldcg(src + static_cast<size_t>(q + u) * p.ss_ld);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += x[u];  // tile order
          }
          for (; q < J.ss_parts; ++q) acc += __ldcg(src + static_cast<size_t>(q) * p.ss_ld);
          s_rs[t] = rsqrtf(acc * J.inv_h + J.eps);
        }
      }
      if (mode == EPI_QKV_ROPE || new_rs) named_bar_sync(2, kEpiThreads);
      if (lane == 0) {
        if (ring)
          mbar_wait(&tfull[seg & 1], (seg >> 1) & 1);
        else
          mbar_wait(&tfull[buf], use & 1);
      }
      __syncwarp();
      tc_fence_after();
      unsigned long long* tre = (p.trace && rank == 0 && et == 0 && seg < kChainTraceSegs)
                                    ? p.trace + (static_cast<size_t>(pair) * kChainTraceSegs + seg) * 8
                                    : nullptr;
      if (tre) tre[3] = globaltimer_ns();
      const uint32_t trow = tmem + ((quarter * 32u) << 16);
      auto scale = [&](int ch, float (&v)[16]) {
        if (scaled) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] *= s_rs[min(ch * 16 + j, tvalid - 1)];
        }
      };
      // split whole-tile job: contributors reduce into a scratch slab, the last one finishes the tile
      const int need = (mode != EPI_ADD_F32 && J.fin_need) ? __ldg(J.fin_need + sg.pt) : 1;
      const bool split = need > 1;
      const int scol = split ? __ldg(J.slab + sg.pt) * 2 * kBM + static_cast<int>(rank) * kBM + static_cast<int>(quarter) * 32 : 0;
      bool last = true;
      if (split) {
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          s_last = atomicAdd(J.arrive + mt, 1) == need - 1;
          if (s_last) {  // every other contributor arrived; wait until their reductions completed
            const unsigned long long t0 = globaltimer_ns();
            while (static_cast<int>(ld_acquire_gpu(reinterpret_cast<const unsigned*>(J.written + mt))) < need - 1) {
              __nanosleep(32);
              if (globaltimer_ns() - t0 > 4000000000ull) __trap();
            }
            J.arrive[mt] = 0;  // re-arm for the next launch
            J.written[mt] = 0;
          }
        }
        named_bar_sync(1, kEpiThreads);
        last = s_last;
        if (last) fence_proxy_async_global();  // the others' bulk reductions -> this CTA's TMA loads
      }
      if (eh >= nchunks) {
        release_tmem();
      } else if (mode == EPI_ADD_F32 || !last) {
        // light epilogue: two chunks in flight per TMEM wait
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
          // token-major 16 x 32 block into the warp's transpose buffer (alternating two), then
          // one bulk reduce-add into h; a buffer is rewritten only after its previous read completed
          auto put = [&](int c, const uint32_t (&r)[16]) {
            float* b = red_par ? sbuf2 : sbuf;
            if (lane == 0) bulk_wait_read1();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; ++j) b[j * 32 + lane] = __uint_as_float(r[j]);
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0 && mt * kBM < J.M) {
              if (split)
                tma_reduce_add_2d(&maps.scr, b, scol, c * 16);
              else
                tma_reduce_add_2d(&maps.hred, b, mt * kBM + static_cast<int>(quarter) * 32, c * 16);
              bulk_commit();
            }
            red_par ^= 1;
          };
          put(ch, ra);
          if (ch + NEH < nchunks) put(ch + NEH, rb);
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
      } else {
        // heavy epilogue (activation / RoPE): the next chunk in flight while this one is emitted;
        // the last contributor of a split tile also streams the other contributors' sum of each
        // chunk (16 tokens x its 32 rows) from the scratch slab into its transpose buffers by TMA
        // (one 2 KB buffer per warp, sbuf2: a chunk's sum is read into registers before the next
        // chunk's load is issued into it; the epilogue itself transposes through sbuf)
        auto fetch = [&](int c) {
          uint64_t* bb = &sbar[ew * 2];
          if (elect_one()) {
            mbar_arrive_expect_tx(bb, 16 * 32 * 4);
            tma_load_2d(sbuf2, &maps.scr, bb, scol, c * 16, policy_evict_first());
          }
          __syncwarp();
        };
        if (split) fetch(eh);
        for (int ch = eh; ch < nchunks; ch += NEH) {
          uint32_t raw[16];
          tmem_ld_32x32b_x16(trow + tcol(ch), raw);
          tmem_ld_wait_regs(raw);
          after_load(ch);
          const bool more = ch + NEH < nchunks;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]);
          if (split) {
            mbar_wait(&sbar[ew * 2], sph[0]);
            sph[0] ^= 1;
            float* zrow = p.scr + static_cast<size_t>(ch * 16) * p.scr_ld + scol + lane;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              v[j] += sbuf2[j * 32 + lane];
              if (ch * 16 + j < tvalid) zrow[static_cast<size_t>(j) * p.scr_ld] = 0.f;  // re-zero the slab
            }
            __syncwarp();
            if (more) fetch(ch + NEH);
          }
          scale(ch, v);
          if (mode == EPI_QKV_ROPE)
            epi_emit<EPI_QKV_ROPE, false>(J.M, p.bn, ep, v, quarter, lane, mt, 0, ch * 16, tvalid, sbuf, s_pos, s_slot,
                                          s_consec, ql);
          else
            epi_emit<FFN, false>(J.M, p.bn, ep, v, quarter, lane, mt, 0, ch * 16, tvalid, sbuf, s_pos, s_slot, s_consec,
                                 ql);
        }
      }
      if (tre) tre[7] = globaltimer_ns();
      // ---- publish ----
      const bool in_range = mt * kBM < J.M;
      if (mode == EPI_ADD_F32 || !last) {  // the bulk reductions of this segment are complete in global memory
        if (lane == 0) bulk_wait0();
        __syncwarp();
        fence_proxy_async_global();
      }
      if (!last) {  // split tile, not the last contributor: publish "my partial is in the slab"
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) atomicAdd(J.written + mt, 1);
      }
      if (mode == EPI_ADD_F32 && J.fin_cnt) {
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          const int old = atomicAdd(J.fin_cnt + mt, 1);
          s_last = old == __ldg(J.fin_need + sg.pt) - 1;
          if (s_last) J.fin_cnt[mt] = 0;  // every contributor arrived: re-arm for the next launch
        }
        named_bar_sync(1, kEpiThreads);
        if (s_last && in_range) {
          __threadfence();
          // finalise 128 columns: X' = bf16(g * h) and the per-token sum of squares (one warp per
          // 16-token block, 4 columns per lane, all 16 loads in flight; a transpose-reduction leaves
          // token u's sum in lanes 2u, 2u+1 after 16 shuffles)
          const float* hsrc = static_cast<const float*>(ep.out);
          const int c0 = mt * kBM + static_cast<int>(lane) * 4;
          const uint2 graw = __ldg(reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(J.fin_g) + c0));
          const float2 g01 = unpack_bf16x2(graw.x), g23 = unpack_bf16x2(graw.y);
          __nv_bfloat16* xa = static_cast<__nv_bfloat16*>(J.fin_xa);
          for (int t0 = ew * 16; t0 < tvalid; t0 += 8 * 16) {
            float4 x[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
              x[u] = t0 + u < tvalid ? __ldcg(reinterpret_cast<const float4*>(hsrc + static_cast<size_t>(t0 + u) * ep.ldo + c0))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            float r[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              r[u] = x[u].x * x[u].x + x[u].y * x[u].y + x[u].z * x[u].z + x[u].w * x[u].w;
              if (t0 + u < tvalid) {
                uint2 pk;
                pk.x = pack_bf16x2(g01.x * x[u].x, g01.y * x[u].y);
                pk.y = pack_bf16x2(g23.x * x[u].z, g23.y * x[u].w);
                *reinterpret_cast<uint2*>(xa + static_cast<size_t>(t0 + u) * J.M + c0) = pk;
              }
            }
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1) {  // offsets 16, 8, 4, 2: keep half of the values
              const bool hi = (lane & (2 * w)) != 0;
#pragma unroll
              for (int i = 0; i < w; ++i) {
                const float keep = hi ? r[i + w] : r[i], send = hi ? r[i] : r[i + w];
                r[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * w);
              }
            }
            r[0] += __shfl_xor_sync(0xffffffffu, r[0], 1);
            const int u = static_cast<int>(lane >> 1);
            if ((lane & 1) == 0 && t0 + u < tvalid) J.fin_ss[static_cast<size_t>(mt) * p.ss_ld + t0 + u] = r[0];
          }
          fence_proxy_async_global();
          __threadfence();
          named_bar_sync(1, kEpiThreads);
          if (et == 0) st_release_gpu(J.flag_out + mt, p.epoch);
        }
      } else if (J.flag_out && last) {
        fence_proxy_async_global();
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0 && in_range) st_release_gpu(J.flag_out + mt, p.epoch);
      }
      if (tre) tre[4] = globaltimer_ns();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (p.span_end && threadIdx.x == 0) atomicMax(p.span_end, globaltimer_ns());
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, p.tmem_cols);
  }
}

uint32_t pow2_cols_c(int n) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(n)) c <<= 1;
  return c;
}

}  // namespace

bool plan_chain_tiling(int N, ChainLaunch* cl) {
  const TokenTiling tt = gemm_token_tiling(N);
  if (tt.n_tiles != 1) return false;
  cl->N = N;
  cl->bn = tt.bn;
  cl->n_mma = tt.n_mma;
  cl->nbuf = tt.bn <= 256 ? 2 : 1;
  const int ni = tt.bn / tt.n_mma;
  const bool ring = tt.n_mma == 2 && 3 * ni <= 512;
  cl->tmem_cols = (cl->nbuf == 2 || ring) ? 512 : pow2_cols_c(tt.bn);
  const size_t stage = kABytes + static_cast<size_t>(tt.bn / 2) * kBK * 2;
  const size_t budget = 226 * 1024 - 1024 - chain_extra_smem(tt.bn);
  cl->stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(8, budget / stage)));
  cl->ring_bytes = static_cast<uint32_t>(cl->stages * stage);
  cl->smem = cl->stages * stage + chain_extra_smem(tt.bn) + 1024;
  return true;
}

cudaError_t launch_chain(const ChainMaps& maps, const ChainLaunch& cl, int ffn_mode, cudaStream_t stream) {
  using KFn = void (*)(const ChainMaps, const ChainLaunch);
  static const KFn fns[2] = {gemm_chain_pair<EPI_SILU_MUL>, gemm_chain_pair<EPI_GELU>};
  static bool configured = false;
  if (!configured) {
    for (KFn fn : fns) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
      if (e != cudaSuccess) return e;
      prefer_max_smem(fn);
    }
    configured = true;
  }
  if (cl.njobs < 1 || cl.njobs > kChainMaxJobs || cl.pairs < 1) return cudaErrorInvalidValue;
  const KFn fn = fns[ffn_mode == EPI_GELU ? 1 : 0];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * cl.pairs);
  cfg.blockDim = dim3(threads_of<kNEHc>());
  cfg.dynamicSmemBytes = cl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  static const bool kbasm_on = !(getenv("SARATHI_GEMM_KBASM") && atoi(getenv("SARATHI_GEMM_KBASM")) == 0);
  static const bool relaxed_on = !(getenv("SARATHI_GEMM_RELAXED") && atoi(getenv("SARATHI_GEMM_RELAXED")) == 0);
  ChainLaunch c2 = cl;
  c2.kbasm = kbasm_on ? 1 : 0;
  c2.relaxed = relaxed_on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, maps, c2);
}

}  // namespace sarathi

// Shared device helpers for the sm_100a kernels: mbarrier, TMA (cp.async.bulk.tensor),
// tcgen05 (UMMA issue, TMEM alloc / ld), bf16 packing.  Raw PTX, no CUTLASS.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda.h>

#define SARATHI_DEVICE __device__ __forceinline__

namespace sarathi {

// ---------------------------------------------------------------------------
// Generic
// ---------------------------------------------------------------------------
SARATHI_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SARATHI_DEVICE uint32_t lane_id() { return threadIdx.x & 31; }

SARATHI_DEVICE unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}

SARATHI_DEVICE uint32_t warp_id_uniform() {
  return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

SARATHI_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

SARATHI_DEVICE uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

SARATHI_DEVICE float2 unpack_bf16x2(uint32_t v) {
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(b);
}

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream serialization
// may start while its predecessor drains; griddep_wait() blocks until the predecessor grid has
// completed and its memory is visible (a no-op without a programmatic dependency);
// griddep_launch_dependents() lets the successor grid start launching.
SARATHI_DEVICE void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
SARATHI_DEVICE void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

SARATHI_DEVICE void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------
SARATHI_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

SARATHI_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

SARATHI_DEVICE void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

SARATHI_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SARATHI_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

SARATHI_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// Wait with cluster-scope acquire (the phase was completed by a remote CTA's release arrive).
SARATHI_DEVICE void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------------------
// TMA (tensor maps are __grid_constant__ kernel parameters)
// ---------------------------------------------------------------------------
SARATHI_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2D tile load; coordinates are (inner, outer) in elements; completion on `bar` (complete_tx).
SARATHI_DEVICE void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

// Plain 1D bulk copy global -> shared (contiguous bytes, multiple of 16, 16-B aligned).
SARATHI_DEVICE void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                 uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(cache_hint)
      : "memory");
}

// L2 cache-policy descriptors (createpolicy).
SARATHI_DEVICE uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
SARATHI_DEVICE uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------------------
// tcgen05 / TMEM
// ---------------------------------------------------------------------------
// Whole warp executes.  Writes the allocated TMEM base address into *holder (shared).
SARATHI_DEVICE void tmem_alloc(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(holder)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

SARATHI_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols)
               : "memory");
}

SARATHI_DEVICE void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
SARATHI_DEVICE void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate), one CTA.
SARATHI_DEVICE void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Warp-uniform variants: the WHOLE warp executes them (operands warp-uniform, so they stay in
// uniform registers); one elected lane issues the instruction.  Avoids the R2UR/ELECT waterfall
// the compiler emits for tcgen05 ops inside a divergent `if (lane == 0)` (~300 cycles per MMA).
SARATHI_DEVICE void umma_f16_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A operand from TMEM (lanes = the M rows, 32-bit columns holding two consecutive bf16 K elements,
// K-major), B from shared memory.
SARATHI_DEVICE void umma_f16_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Eight k16 UMMAs (cta_group::1) in ONE asm block with one elect (see umma_kblock_ss_pair for why):
// both operands in shared memory, the descriptor of step k = desc0 + (k / 4) * half + (k % 4) * 2
// (a 128-deep K split in two 64-element SW128 halves, 32 B per k16 step).  acc0: accumulate at k = 0.
SARATHI_DEVICE void umma8_ss_halves(uint32_t d, uint64_t a0, uint64_t ah, uint64_t b0, uint64_t bh, uint32_t idesc,
                                    uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a<8>, b<8>;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 q, %6, %6;\n\t"
      "mov.b64 a0, %1;\n\tadd.s64 a1, a0, 2;\n\tadd.s64 a2, a0, 4;\n\tadd.s64 a3, a0, 6;\n\t"
      "add.s64 a4, a0, %2;\n\tadd.s64 a5, a4, 2;\n\tadd.s64 a6, a4, 4;\n\tadd.s64 a7, a4, 6;\n\t"
      "mov.b64 b0, %3;\n\tadd.s64 b1, b0, 2;\n\tadd.s64 b2, b0, 4;\n\tadd.s64 b3, b0, 6;\n\t"
      "add.s64 b4, b0, %4;\n\tadd.s64 b5, b4, 2;\n\tadd.s64 b6, b4, 4;\n\tadd.s64 b7, b4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %5, q;\n\t}\n" ::"r"(d),
      "l"(a0), "l"(ah), "l"(b0), "l"(bh), "r"(idesc), "r"(acc0)
      : "memory");
}
// Eight k16 UMMAs (cta_group::1) in one asm block, A from TMEM at t0 + (k / 4) * 64 + (k % 4) * 8
// (packed bf16 pairs, two 64-column halves), B descriptor(k) = b0 + k * bstep.
SARATHI_DEVICE void umma8_ts(uint32_t d, uint32_t t0, uint64_t b0, uint64_t bstep, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b64 b<8>;\n\t.reg .b32 t<8>;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 q, %5, %5;\n\t"
      "mov.b32 t0, %1;\n\tadd.u32 t1, t0, 8;\n\tadd.u32 t2, t0, 16;\n\tadd.u32 t3, t0, 24;\n\t"
      "add.u32 t4, t0, 64;\n\tadd.u32 t5, t0, 72;\n\tadd.u32 t6, t0, 80;\n\tadd.u32 t7, t0, 88;\n\t"
      "mov.b64 b0, %2;\n\tadd.s64 b1, b0, %3;\n\tadd.s64 b2, b1, %3;\n\tadd.s64 b3, b2, %3;\n\t"
      "add.s64 b4, b3, %3;\n\tadd.s64 b5, b4, %3;\n\tadd.s64 b6, b5, %3;\n\tadd.s64 b7, b6, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t0], b0, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t4], b4, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t5], b5, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t6], b6, %4, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t7], b7, %4, q;\n\t}\n" ::"r"(d),
      "r"(t0), "l"(b0), "l"(bstep), "r"(idesc), "r"(acc0)
      : "memory");
}
SARATHI_DEVICE void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread completed.
SARATHI_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread.
SARATHI_DEVICE void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

SARATHI_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

SARATHI_DEVICE void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
SARATHI_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// wait::ld that also "defines" r: the registers of an in-flight tcgen05.ld must not be read (or
// copied) by compiled code before the wait, so they are tied to it as read-write operands.
SARATHI_DEVICE void tmem_ld_wait_regs(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

// UMMA shared-memory matrix descriptor, K-major operand, 128-byte swizzle:
//   start address >> 4 in [0,14), LBO (ignored for swizzled K-major, 1) in [16,30),
//   SBO = 1024 B (8 rows x 128 B) >> 4 in [32,46), version 1 in [46,48), layout 2 (SW128) in [61,64).
SARATHI_DEVICE uint64_t make_desc_k_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// ---------------------------------------------------------------------------
// Clusters and the CTA pair (cta_group::2)
// ---------------------------------------------------------------------------
SARATHI_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

SARATHI_DEVICE void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// shared::cta address -> shared::cluster address of the same offset in CTA `rank`.
SARATHI_DEVICE uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

SARATHI_DEVICE void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// Relaxed remote arrive for TMEM-slot releases: the waiter (the MMA issuer) needs only the
// arriving warp's completed tcgen05.ld (ordered by tcgen05.wait::ld + tcgen05.fence::before_thread_sync),
// not its generic global stores; .release.cluster compiles to MEMBAR.ALL.GPU, which waits for every
// store / red.add the epilogue warp has in flight before the slot is handed back.
SARATHI_DEVICE void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

// Pair TMA load: data lands in this CTA's smem, transaction bytes are counted on the LEADER's
// (rank 0) mbarrier (peer bit of the barrier address cleared).
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
SARATHI_DEVICE void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                     uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

// Warp-uniform pair TMA / expect_tx (whole warp executes, one elected lane issues).
SARATHI_DEVICE void tma_load_2d_pair_warp(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                          uint64_t cache_hint) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

// Warp-uniform single-CTA 2D TMA load (one elected lane issues).
SARATHI_DEVICE void tma_load_2d_warp(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

SARATHI_DEVICE void mbar_arrive_expect_tx_warp(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

SARATHI_DEVICE void tmem_alloc_pair(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(holder)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}

SARATHI_DEVICE void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A * B^T over the CTA pair: M = 256 (128 rows of A from each CTA), the N columns of B
// split in halves across the two CTAs' smem at the same offsets.  Issued by the leader only.
SARATHI_DEVICE void umma_f16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

SARATHI_DEVICE void umma_f16_ss_pair_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Pair MMA with the A operand from TMEM (each CTA's 128 rows at the same TMEM address; lanes = rows,
// 32-bit columns holding two consecutive bf16 K elements), B from shared memory.
SARATHI_DEVICE void umma_f16_ts_pair_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One 64-deep k-block of pair MMAs (4 k16 steps; per step UMMA 0 into d0 and, if `two`, UMMA 1 into
// d1 over the second B slice) issued by ONE elected lane in ONE asm block.  The k16 slices advance
// the SW128 K-major descriptors by 32 B (+2 in the 16-B address field) and the TMEM A operand by 8
// columns.  Issuing each UMMA through its own asm statement cost ~20 SASS instructions per UMMA
// (ELECT, R2UR.BROADCAST x5, VOTEU, BRA.DIV): at <= 256 tokens the issue, not the tensor core,
// paced the k-block (tools/experiments.sh narrow2: 0.34 us per k-block at N = 144 with no loads at all).
// acc0: accumulate into d for the first k16 step (the later steps always accumulate).
SARATHI_DEVICE void umma_kblock_ss_pair(uint32_t d0, uint32_t d1, uint64_t a_desc, uint64_t b_desc0, uint64_t b_desc1,
                                        uint32_t idesc0, uint32_t idesc1, uint32_t acc0, uint32_t two) {
  asm volatile(
      "{\n\t.reg .pred e, t, p, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, c1, c2, c3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %7, 0;\n\t"
      "setp.eq.b32 q, %7, %7;\n\t"
      "setp.ne.and.b32 t, %8, 0, e;\n\t"
      "add.s64 a1, %2, 2;\n\tadd.s64 a2, %2, 4;\n\tadd.s64 a3, %2, 6;\n\t"
      "add.s64 b1, %3, 2;\n\tadd.s64 b2, %3, 4;\n\tadd.s64 b3, %3, 6;\n\t"
      "add.s64 c1, %4, 2;\n\tadd.s64 c2, %4, 4;\n\tadd.s64 c3, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, p;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %5, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], a1, c1, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %5, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], a2, c2, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %5, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], a3, c3, %6, q;\n\t}\n" ::"r"(d0),
      "r"(d1), "l"(a_desc), "l"(b_desc0), "l"(b_desc1), "r"(idesc0), "r"(idesc1), "r"(acc0), "r"(two)
      : "memory");
}
// The same with the A operand staged into TMEM first (tcgen05.cp of each k16 slice to a_tmem + 8k;
// cp and mma execute in issue order), both UMMAs reading A from TMEM.
SARATHI_DEVICE void umma_kblock_ts_pair(uint32_t d0, uint32_t d1, uint32_t a_tmem, uint64_t a_sdesc, uint64_t b_desc0,
                                        uint64_t b_desc1, uint32_t idesc0, uint32_t idesc1, uint32_t acc0, uint32_t two) {
  asm volatile(
      "{\n\t.reg .pred e, t, p, q;\n\t.reg .b64 s1, s2, s3, b1, b2, b3, c1, c2, c3;\n\t.reg .b32 t1, t2, t3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "setp.eq.b32 q, %8, %8;\n\t"
      "setp.ne.and.b32 t, %9, 0, e;\n\t"
      "add.s64 s1, %3, 2;\n\tadd.s64 s2, %3, 4;\n\tadd.s64 s3, %3, 6;\n\t"
      "add.s64 b1, %4, 2;\n\tadd.s64 b2, %4, 4;\n\tadd.s64 b3, %4, 6;\n\t"
      "add.s64 c1, %5, 2;\n\tadd.s64 c2, %5, 4;\n\tadd.s64 c3, %5, 6;\n\t"
      "add.u32 t1, %2, 8;\n\tadd.u32 t2, %2, 16;\n\tadd.u32 t3, %2, 24;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [%2], %3;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %4, %6, p;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], [%2], %5, %7, p;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [t1], s1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t1], b1, %6, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], [t1], c1, %7, q;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [t2], s2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t2], b2, %6, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], [t2], c2, %7, q;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [t3], s3;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t3], b3, %6, q;\n\t"
      "@t tcgen05.mma.cta_group::2.kind::f16 [%1], [t3], c3, %7, q;\n\t}\n" ::"r"(d0),
      "r"(d1), "r"(a_tmem), "l"(a_sdesc), "l"(b_desc0), "l"(b_desc1), "r"(idesc0), "r"(idesc1), "r"(acc0), "r"(two)
      : "memory");
}
// shared memory -> TMEM copy of a 128-row x 256-bit matrix (one k16 slice of a K-major bf16 operand)
// in both CTAs of the pair (each from its own shared memory); executes in issue order with the MMAs
SARATHI_DEVICE void tmem_cp_128x256b_pair_warp(uint32_t taddr, uint64_t s_desc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [%0], %1;\n\t}\n" ::"r"(taddr),
      "l"(s_desc)
      : "memory");
}
SARATHI_DEVICE void umma_commit_pair_mc_warp(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// Arrive on the mbarrier at this smem offset in every CTA of `cta_mask` once all prior pair MMAs
// issued by this thread completed.
SARATHI_DEVICE void umma_commit_pair_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// Instruction descriptor for kind::f16: D fp32, A/B bf16, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t make_idesc_bf16_f32(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format = F32
         | (1u << 7)          // a_format = BF16
         | (1u << 10)         // b_format = BF16
         | (0u << 15)         // a K-major
         | (0u << 16)         // b K-major
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

// Host: launch with programmatic stream serialization (PDL) unless SARATHI_PDL=0.
bool pdl_enabled();
// Host: every kernel of the layer chain prefers the maximum shared-memory carveout, so an SM does
// not switch its L1 / shared split between a 226-KB GEMM CTA and a small RMSNorm CTA at every kernel
// boundary (SARATHI_CARVEOUT=0 leaves the driver's default).  Idempotent per kernel.
bool carveout_enabled();
template <typename... KArgs>
void prefer_max_smem(void (*kernel)(KArgs...)) {
  if (carveout_enabled())
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  static bool carved = false;  // one flag per kernel instantiation of this template
  if (!carved) {
    prefer_max_smem(kernel);
    carved = true;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace sarathi

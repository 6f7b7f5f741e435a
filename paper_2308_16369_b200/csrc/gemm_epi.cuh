// Device pieces shared by the tcgen05 GEMM kernels (gemm.cu: one GEMM per launch;
// gemm_chain.cu: the layer chain): tile constants, activations and the fused epilogues.
#pragma once

#include "common.cuh"
#include "gemm.cuh"

namespace sarathi {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
// warp 0 TMA, warp 1 MMA, warps 2 .. 2 + 4*NEH - 1 epilogue (NEH warps per TMEM lane quarter)
template <int NEH>
constexpr int threads_of() { return 64 + 128 * NEH; }
constexpr int kWRowsPerTile = 32;            // packed W viewed as rows of 256 elements (512 B)

SARATHI_DEVICE float silu_f(float x) { return __fdividef(x, 1.0f + __expf(-x)); }
SARATHI_DEVICE float gelu_tanh_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(k0 * (x + k1 * x * x * x)));  // |err| ~ 2^-11, below bf16 output ulp
  return 0.5f * x * (1.0f + t);
}

// ---------------------------------------------------------------------------
// Epilogue.  The accumulator comes out of TMEM with thread = row (tcgen05.ld 32x32b: lane l of
// warp quarter q holds row 32q + l of this CTA's 128-row tile) and registers = 16 consecutive
// tokens.  Outputs are token-major ([token][feature]), so each warp transposes its 32 x 16 block
// through a private 2 KB shared-memory buffer and writes 16-byte vectors (8 bf16 / 4 fp32 features
// of one token) — the residual add is a vector red.global.add.v4.f32.  No cross-warp barrier.
//
// Row orders the packed weights are generated in (host_sched.cpp shard_map) so that every fused
// epilogue is warp-local:
//  * gate||up (SwiGLU): 16-row interleave — packed rows [32b, 32b+16) = gate features
//    [16b, 16b+16), rows [32b+16, 32b+32) = the matching up features; lane l and l^16 of a warp
//    hold g and u of the same feature (one shuffle).
//  * QKV: inside each head, warp-slab j (rows 32j..32j+31 of the head) holds dims
//    [16j, 16j+16) in lanes 0-15 and their rotate-half partners [hd/2 + 16j, ...) in lanes 16-31,
//    so RoPE is one shuffle.  Q, K and V are stored in the natural dim order.
// ---------------------------------------------------------------------------
constexpr int kStageFloats = 16 * 32;  // per-warp transpose buffer (2 KB)

// RoPE angles are computed in registers (no table traffic: table loads from the epilogue cost an
// L2/HBM round trip per 16-token chunk and dominated the QKV GEMM).  angle = pos * theta_i with
// theta_i = base^(-2i/hd) held as an fp32 pair (hi + lo, from fp64 on the host), the product kept
// exact with an FMA, reduced mod 2*pi by a 3-constant Cody-Waite step, then __sincosf on |r| <= pi
// (abs error ~2^-21; angle error <= 2.3e-7 rad for pos <= 2e5, checked against fp64).
SARATHI_DEVICE void rope_cos_sin(int pos, float th_hi, float th_lo, float& c, float& s) {
  const float p = static_cast<float>(pos);
  const float a_hi = p * th_hi;
  const float a_lo = fmaf(p, th_hi, -a_hi) + p * th_lo;
  const float k = rintf(a_hi * 0.15915494309189535f);  // round(a / 2pi)
  float r = fmaf(-k, 6.28125f, a_hi);                   // 2pi = 6.28125 + 1.9353071795864769e-3 + ...
  r = fmaf(-k, 1.9353071795864769e-3f, r);
  r = fmaf(-k, 1.0253132e-11f, r);  // 2pi - 6.28125 - fp32(1.9353071795864769e-3)
  r += a_lo;
  __sincosf(r, &s, &c);
}

struct QkvLane {  // per-warp / per-lane constants of the fused QKV epilogue
  int gh;         // packed head index in [q heads | k heads | v heads]
  int jw;         // warp slab within the head
  int dd;         // rotation index of this lane (dim within the half)
  bool rope;      // q or k head
  float th_hi, th_lo;  // theta_dd = base^(-2 dd / hd) as hi + lo
  float cd, sd;        // cos / sin of one position step (theta_dd): the consecutive-position recurrence
};

SARATHI_DEVICE QkvLane qkv_lane(const EpiParams& ep, int mt, uint32_t q, uint32_t lane) {
  QkvLane o;
  const int hd_shift = ep.head_dim == 128 ? 7 : 6;
  const int row0 = mt * kBM + static_cast<int>(q) * 32;
  o.gh = row0 >> hd_shift;
  o.jw = (row0 & (ep.head_dim - 1)) >> 5;
  o.dd = 16 * o.jw + static_cast<int>(lane & 15);
  o.rope = o.gh < ep.n_q_local + ep.n_kv_local;
  o.th_hi = __ldg(ep.rope_theta + 2 * o.dd);
  o.th_lo = __ldg(ep.rope_theta + 2 * o.dd + 1);
  rope_cos_sin(1, o.th_hi, o.th_lo, o.cd, o.sd);
  return o;
}

// Orders later uses of r after a preceding tcgen05.wait::ld (a second in-flight load's registers).
SARATHI_DEVICE void regs_fence(uint32_t (&r)[16]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

SARATHI_DEVICE void red_add_v4(float* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int MODE, bool DBG>
SARATHI_DEVICE void epi_emit(const int M, const int bn, const EpiParams& ep, float (&v)[16], uint32_t q, uint32_t lane, int mt,
                             int nt, int c0, int tvalid, float* sbuf, const int* s_pos, const int* s_slot,
                             const int* s_consec, const QkvLane& ql, unsigned long long* trc = nullptr) {
  const int row0 = mt * kBM + static_cast<int>(q) * 32;  // first accumulator row of this warp
  const long long tb = static_cast<long long>(nt) * bn + c0;
  const int nv = (DBG && (ep.dbg & 8)) ? 0 : min(16, tvalid - c0);  // dbg bit 3: no global stores
  uint16_t* sb = reinterpret_cast<uint16_t*>(sbuf);
  switch (MODE) {
    case EPI_STORE_BF16:
    case EPI_GELU: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float x = MODE == EPI_GELU ? gelu_tanh_f(v[j]) : v[j];
        sb[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(x));
      }
      __syncwarp();
      const int g = static_cast<int>(lane & 3), m = row0 + g * 8;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int tok = pass * 8 + static_cast<int>(lane >> 2);
        if (tok < nv && m < M)
          *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + (tb + tok) * ep.ldo + m) =
              *reinterpret_cast<const uint4*>(sb + tok * 32 + g * 8);
      }
      __syncwarp();
      break;
    }
    case EPI_STORE_F32:
    case EPI_ADD_F32: {
#pragma unroll
      for (int j = 0; j < 16; ++j) sbuf[j * 32 + lane] = v[j];
      __syncwarp();
      const int g = static_cast<int>(lane & 7), m = row0 + g * 4;
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int tok = pass * 4 + static_cast<int>(lane >> 3);
        if (tok < nv && m < M) {
          const float4 x = *reinterpret_cast<const float4*>(sbuf + tok * 32 + g * 4);
          float* dst = static_cast<float*>(ep.out) + (tb + tok) * ep.ldo + m;
          if (MODE == EPI_ADD_F32)
            red_add_v4(dst, x);
          else
            *reinterpret_cast<float4*>(dst) = x;
        }
      }
      __syncwarp();
      break;
    }
    case EPI_SILU_MUL: {
      // lanes 0-15: gate of features f0 + (l & 15); lanes 16-31: up of the same features.
      // After one xor-16 exchange lanes 0-15 own tokens 0-7 and lanes 16-31 tokens 8-15.
      const bool lo = lane < 16;
      const int f0 = row0 >> 1;  // 16 output features per warp
      float y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = __shfl_xor_sync(0xffffffffu, lo ? v[8 + i] : v[i], 16);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gv = lo ? v[i] : y[i], uv = lo ? y[i] : v[8 + i];
        sb[((lo ? 0 : 8) + i) * 16 + (lane & 15)] = __bfloat16_as_ushort(__float2bfloat16_rn(silu_f(gv) * uv));
      }
      __syncwarp();
      const int tok = static_cast<int>(lane >> 1), h8 = static_cast<int>(lane & 1) * 8;
      if (tok < nv && row0 < M)
        *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + (tb + tok) * ep.ldo + f0 + h8) =
            *reinterpret_cast<const uint4*>(sb + tok * 16 + h8);
      __syncwarp();
      break;
    }
    case EPI_QKV_ROPE: {
      const int half = ep.head_dim >> 1;
      const bool lo = lane < 16;
      if (ql.rope && !(DBG && (ep.dbg & 32))) {  // dbg bit 5: no RoPE math (timing only)
        // branch-free, 8 tokens per batch so the shuffles, position loads and sincos of different
        // tokens overlap (a per-token dependent chain cost ~150 cycles x 16 per chunk)
        // consecutive positions (prefill chunks): angle-addition recurrence from the chunk's first
        // position, 4 FMAs per token instead of a reduction + sincos (error growth ~16 ulp)
        const bool consec = s_consec[c0 >> 4] != 0;
        const float cd = ql.cd, sd = ql.sd;
        float cr = 1.f, sr = 0.f;
        if (consec) rope_cos_sin(s_pos[c0], ql.th_hi, ql.th_lo, cr, sr);
#pragma unroll
        for (int j0 = 0; j0 < 16; j0 += 8) {
          float xp[8], c[8], sn[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) xp[j] = __shfl_xor_sync(0xffffffffu, v[j0 + j], 16);  // rotate-half partner
          if (consec) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              c[j] = cr;
              sn[j] = sr;
              const float cn = fmaf(cr, cd, -sr * sd);
              sr = fmaf(sr, cd, cr * sd);
              cr = cn;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) rope_cos_sin(s_pos[min(c0 + j0 + j, tvalid - 1)], ql.th_hi, ql.th_lo, c[j], sn[j]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            // x1 = low-half value, x2 = high-half value: y1 = x1 c - x2 s, y2 = x2 c + x1 s
            const float y = lo ? v[j0 + j] * c[j] - xp[j] * sn[j] : v[j0 + j] * c[j] + xp[j] * sn[j];
            sb[(j0 + j) * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(y));
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) sb[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(v[j]));
      }
      __syncwarp();
      if (trc && lane == 0) *trc = globaltimer_ns();
      if (row0 < M) {
        const int hd_shift = ep.head_dim == 128 ? 7 : 6;
        const bool isq = ql.gh < ep.n_q_local;
        const int kvh = isq ? 0 : (ql.rope ? ql.gh - ep.n_q_local : ql.gh - ep.n_q_local - ep.n_kv_local);
        __nv_bfloat16* cache = static_cast<__nv_bfloat16*>(ql.rope ? ep.kcache : ep.vcache);
        const int g = static_cast<int>(lane & 3);  // 8-dim group: 0,1 low half; 2,3 high half
        const int d = (g < 2 ? 0 : half) + 16 * ql.jw + (g & 1) * 8;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int tok = pass * 8 + static_cast<int>(lane >> 2);
          if (tok >= nv || (DBG && (ep.dbg & 16) && !isq)) continue;  // dbg bit 4: no K/V cache stores
          __nv_bfloat16* dst =
              isq ? static_cast<__nv_bfloat16*>(ep.out) + (tb + tok) * ep.ldo + (ql.gh << hd_shift) + d
                  : cache + (static_cast<size_t>(s_slot[c0 + tok] + kvh * ep.block_size) << hd_shift) + d;
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(sb + tok * 32 + g * 8);
        }
      }
      __syncwarp();
      break;
    }
    default:
      break;
  }
}

}  // namespace
}  // namespace sarathi

"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no norm, no attention, no
matmul, no scheduling).  It only defines:

* the model configurations named in BASELINE.json / SURVEY.md §8 (hyper-parameters);
* the counter-based weight / token generator spec (SURVEY.md §8(c) "Weight / input
  generator spec"), implemented here in NumPy.  The CUDA library implements the same
  spec independently (paper_2308_16369_b200/csrc/weightgen.cu); the two share no code;
* the workload generator of the paper's evaluation (Zipf(θ) lengths in [1K, 4K] and the
  per-request P:D split, §5.3), whose random draws come from the same
  counter-based hash.

Generator spec (bit-exact, both sides):
    splitmix64(x):  z = x + 0x9E3779B97F4A7C15
                    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                    return z ^ (z >> 31)                         (all mod 2^64)
    u24(seed, tau, k) = splitmix64(seed ^ (tau << 40 | k)) >> 40          in [0, 2^24)
    v = 2*u24 - (2^24 - 1)                                   odd integer, |v| < 2^24
    weight  = bf16_rne( f32(v) *f32 s ),  s = f32(sqrt(3) * sigma / 2^24)   (one fp32 RNE multiply)
    gain    = bf16_rne( 1.0f +f32 (f32(v) *f32 f32(0.1 / 2^24)) )           (fp32 RNE mul, then add)
    token   = (u24(tok_seed, 2^21 + req_id, pos) * V) >> 24
Flat index k enumerates the LOGICAL (unsharded) tensor, row-major, in PyTorch nn.Linear
layout [out_features, in_features]; a tensor-parallel shard takes rows / columns of it.
"""
from __future__ import annotations

import dataclasses
import math
import os
from typing import Dict, List, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

# ---------------------------------------------------------------------------
# Model configurations (PAPER.md L114 fixes layers / heads / hidden; the rest are the
# readings O-1..O-6 of SURVEY.md §8(c), restated in DESIGN.md).
# ---------------------------------------------------------------------------
FFN_SWIGLU = 0
FFN_GELU = 1


@dataclasses.dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_hidden: int
    vocab: int
    ffn_kind: int = FFN_SWIGLU
    rms_eps: float = 1e-5
    rope_base: float = 10000.0
    max_seq_len: int = 4096

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def with_layers(self, n: int) -> "ModelConfig":
        return dataclasses.replace(self, n_layers=n, name=f"{self.name}-L{n}")

    def params_per_layer(self) -> int:
        H, H2 = self.hidden, self.ffn_hidden
        attn = H * (self.q_dim + 2 * self.kv_dim) + self.q_dim * H
        ffn = (3 if self.ffn_kind == FFN_SWIGLU else 2) * H * H2
        return attn + ffn + 2 * H

    def kv_bytes_per_token(self, tp: int = 1) -> int:
        """m_kv of PAPER.md L393 (reading O-18): K and V, all layers, bf16, per GPU."""
        return 2 * self.n_layers * (self.n_kv_heads // tp if self.n_kv_heads >= tp else 1) * self.head_dim * 2


TINY = ModelConfig("tiny", 2, 256, 4, 4, 64, 768, 512, max_seq_len=128)
LLAMA_13B = ModelConfig("llama-13b", 40, 5120, 40, 40, 128, 13824, 32000)
LLAMA_33B = ModelConfig("llama-33b", 60, 6656, 52, 52, 128, 17920, 32000)
LLAMA2_70B = ModelConfig("llama2-70b", 80, 8192, 64, 8, 128, 28672, 32000)
GPT3_175B = ModelConfig("gpt3-175b", 96, 12288, 96, 96, 128, 49152, 50304, ffn_kind=FFN_GELU)
CONFIGS: Dict[str, ModelConfig] = {c.name: c for c in (TINY, LLAMA_13B, LLAMA_33B, LLAMA2_70B, GPT3_175B)}

# ---------------------------------------------------------------------------
# Tensor enumeration and init scales.
# ---------------------------------------------------------------------------
WQ, WK, WV, WO, WG, WU, WD, G1, G2 = range(9)  # per layer: tau = 16*layer + kind
EMB_TAU = 1 << 20
GF_TAU = (1 << 20) + 1
WLM_TAU = (1 << 20) + 2
TOKEN_TAU_BASE = 1 << 21
ZIPF_TAU_BASE = 1 << 22

KIND_NAMES = {WQ: "wq", WK: "wk", WV: "wv", WO: "wo", WG: "wg", WU: "wu", WD: "wd", G1: "g1", G2: "g2"}


def layer_tau(layer: int, kind: int) -> int:
    return 16 * layer + kind


def tensor_shape(cfg: ModelConfig, kind: int) -> Tuple[int, ...]:
    H, H2 = cfg.hidden, cfg.ffn_hidden
    return {
        WQ: (cfg.q_dim, H), WK: (cfg.kv_dim, H), WV: (cfg.kv_dim, H), WO: (H, cfg.q_dim),
        WG: (H2, H), WU: (H2, H), WD: (H, H2), G1: (H,), G2: (H,),
    }[kind]


def tensor_sigma(cfg: ModelConfig, kind: int) -> float:
    """Init std per tensor: 1/sqrt(fan_in); O and down additionally 1/sqrt(2L) (reading O-21)."""
    H, H2 = cfg.hidden, cfg.ffn_hidden
    depth = 1.0 / math.sqrt(2.0 * cfg.n_layers)
    return {
        WQ: 1.0 / math.sqrt(H), WK: 1.0 / math.sqrt(H), WV: 1.0 / math.sqrt(H),
        WO: depth / math.sqrt(cfg.q_dim), WG: 1.0 / math.sqrt(H), WU: 1.0 / math.sqrt(H),
        WD: depth / math.sqrt(H2),
    }[kind]


def weight_scale_f32(sigma: float) -> np.float32:
    return np.float32(math.sqrt(3.0) * sigma / float(1 << 24))


GAIN_SCALE_F32 = np.float32(0.1 / float(1 << 24))

# ---------------------------------------------------------------------------
# Counter-based hash.
# ---------------------------------------------------------------------------


def splitmix64_scalar(x: int) -> int:
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def u24(seed: int, tau: int, k: np.ndarray) -> np.ndarray:
    key = np.uint64((seed ^ (tau << 40)) & MASK64) ^ k.astype(np.uint64)
    return (splitmix64(key) >> np.uint64(40)).astype(np.int64)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even fp32 -> bf16 (finite inputs), returned as uint16 bits."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))
    return (b >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _odd_v(seed: int, tau: int, k: np.ndarray) -> np.ndarray:
    return (2 * u24(seed, tau, k) - ((1 << 24) - 1)).astype(np.float32)


def gen_weight_bits(seed: int, tau: int, sigma: float, start: int, count: int) -> np.ndarray:
    """bf16 bits of flat elements [start, start+count) of a weight tensor."""
    k = np.arange(start, start + count, dtype=np.uint64)
    x = _odd_v(seed, tau, k) * weight_scale_f32(sigma)  # fp32 * fp32 -> fp32 (RNE)
    return f32_to_bf16_bits(x)


def gen_gain_bits(seed: int, tau: int, n: int) -> np.ndarray:
    k = np.arange(n, dtype=np.uint64)
    x = np.float32(1.0) + _odd_v(seed, tau, k) * GAIN_SCALE_F32
    return f32_to_bf16_bits(x.astype(np.float32))


def _chunked_bits(seed: int, tau: int, sigma: float, total: int, chunk: int = 1 << 22) -> np.ndarray:
    """Chunks are independent (counter-based), so they are generated on a thread pool (NumPy
    releases the GIL inside the uint64 ufuncs); the bits do not depend on the chunking."""
    out = np.empty(total, dtype=np.uint16)

    def one(s):
        n = min(chunk, total - s)
        out[s:s + n] = gen_weight_bits(seed, tau, sigma, s, n)

    starts = range(0, total, chunk)
    if total <= chunk:
        one(0)
        return out
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(one, starts))
    return out


def layer_tensor_bits(cfg: ModelConfig, seed: int, layer: int, kind: int) -> np.ndarray:
    """bf16 bits of one logical per-layer tensor, shaped as tensor_shape()."""
    shape = tensor_shape(cfg, kind)
    tau = layer_tau(layer, kind)
    if kind in (G1, G2):
        return gen_gain_bits(seed, tau, shape[0])
    return _chunked_bits(seed, tau, tensor_sigma(cfg, kind), int(np.prod(shape))).reshape(shape)


def layer_tensor_rows_bits(cfg: ModelConfig, seed: int, layer: int, kind: int, rows: Sequence[int]) -> np.ndarray:
    """Selected rows of a per-layer matrix (for sampled checks at full size)."""
    shape = tensor_shape(cfg, kind)
    tau = layer_tau(layer, kind)
    sig = tensor_sigma(cfg, kind)
    out = np.empty((len(rows), shape[1]), dtype=np.uint16)
    for i, r in enumerate(rows):
        out[i] = gen_weight_bits(seed, tau, sig, int(r) * shape[1], shape[1])
    return out


def embedding_rows_bits(cfg: ModelConfig, seed: int, rows: Sequence[int]) -> np.ndarray:
    out = np.empty((len(rows), cfg.hidden), dtype=np.uint16)
    for i, r in enumerate(rows):
        out[i] = gen_weight_bits(seed, EMB_TAU, 1.0, int(r) * cfg.hidden, cfg.hidden)
    return out


def embedding_bits(cfg: ModelConfig, seed: int) -> np.ndarray:
    return _chunked_bits(seed, EMB_TAU, 1.0, cfg.vocab * cfg.hidden).reshape(cfg.vocab, cfg.hidden)


def final_gain_bits(cfg: ModelConfig, seed: int) -> np.ndarray:
    return gen_gain_bits(seed, GF_TAU, cfg.hidden)


def lm_head_bits(cfg: ModelConfig, seed: int) -> np.ndarray:
    return _chunked_bits(seed, WLM_TAU, 1.0 / math.sqrt(cfg.hidden), cfg.vocab * cfg.hidden).reshape(cfg.vocab, cfg.hidden)


def lm_head_rows_bits(cfg: ModelConfig, seed: int, rows: Sequence[int]) -> np.ndarray:
    sig = 1.0 / math.sqrt(cfg.hidden)
    out = np.empty((len(rows), cfg.hidden), dtype=np.uint16)
    for i, r in enumerate(rows):
        out[i] = gen_weight_bits(seed, WLM_TAU, sig, int(r) * cfg.hidden, cfg.hidden)
    return out


def as_f64(bits: np.ndarray) -> np.ndarray:
    """Exact upcast of bf16 bits to float64."""
    return bf16_bits_to_f32(bits).astype(np.float64)


# ---------------------------------------------------------------------------
# Tokens (teacher-forced, reading O-12) and the paper's workload generator.
# ---------------------------------------------------------------------------


def tokens(tok_seed: int, req_id: int, start: int, count: int, vocab: int) -> np.ndarray:
    """Token ids of request req_id at positions [start, start+count)."""
    k = np.arange(start, start + count, dtype=np.uint64)
    u = u24(tok_seed, TOKEN_TAU_BASE + req_id, k)
    return ((u * vocab) >> 24).astype(np.int32)


def u53(seed: int, stream: int, k: np.ndarray) -> np.ndarray:
    key = np.uint64((seed ^ ((ZIPF_TAU_BASE + stream) << 40)) & MASK64) ^ k.astype(np.uint64)
    return (splitmix64(key) >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def zipf_lengths(seed: int, n: int, lo: int = 1024, hi: int = 4096, theta: float = 0.4) -> np.ndarray:
    """n sequence lengths ~ Zipf(theta) over integers [lo, hi], rank 1 = shortest (reading O-19).

    PAPER.md L10-11 (§5.3): "sampled from a Zipf distribution (θ = 0.4)" with min/max 1K/4K.
    """
    ranks = np.arange(1, hi - lo + 2, dtype=np.float64)
    w = ranks ** (-theta)
    cdf = np.cumsum(w) / w.sum()
    u = u53(seed, 0, np.arange(n, dtype=np.uint64))
    idx = np.searchsorted(cdf, u, side="right")
    return (lo + np.minimum(idx, hi - lo)).astype(np.int64)


def split_pd(length: int, pd_ratio: float) -> Tuple[int, int]:
    """P, D for a request of total length with the desired P:D ratio."""
    p = int(round(length * pd_ratio / (1.0 + pd_ratio)))
    p = max(1, min(length - 1, p))
    return p, length - p


@dataclasses.dataclass(frozen=True)
class RequestSpec:
    req_id: int
    prompt_len: int  # P
    decode_len: int  # D
    arrival_iter: int = 0


def zipf_workload(seed: int, n: int, pd_ratio: float, lo: int = 1024, hi: int = 4096,
                  theta: float = 0.4) -> List[RequestSpec]:
    lens = zipf_lengths(seed, n, lo, hi, theta)
    out = []
    for i, ln in enumerate(lens):
        p, d = split_pd(int(ln), pd_ratio)
        out.append(RequestSpec(i, p, d, 0))
    return out

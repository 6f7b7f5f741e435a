"""fp64 transformer forward for the SARATHI hot path — TEST INFRASTRUCTURE ONLY.

The method's claim (§4.2): chunked prefill with the progressive causal mask is
"mathematically equivalent to the full prefill"; linear ops are row-wise so fusing the tokens
of different requests into one matmul changes nothing (§4.3); decode with a KV
cache equals recomputation (§2.2).  Hence the oracle IS the plain definition:

    h_i^0 = E[x_i]
    for l in 1..L:                                  (block of P:L193-203, §2.1; reading O-1)
        a_i   = RMSNorm(h_i^{l-1}; g1_l)
        q,k,v = a_i Wq^T, a_i Wk^T, a_i Wv^T ; RoPE on q,k at position i       (preproj)
        o_i   = sum_{j<=i} softmax_j(q_i.k_j / sqrt(hd)) v_j  (per head, GQA)   (attn)
        u_i   = h_i^{l-1} + o_i Wo^T                                           (postproj)
        b_i   = RMSNorm(u_i; g2_l)
        f_i   = (SiLU(b_i Wg^T) * (b_i Wu^T)) Wd^T     [GELU_tanh(b W1^T) W2^T]  (ffn_ln1/2)
        h_i^l = u_i + f_i
    logits_i = RMSNorm(h_i^L; g_f) Wlm^T

``forward_full`` evaluates it per request over the whole token history with a dense causal
mask.  ``IncrementalOracle`` replays a hybrid-batch schedule step by step in the paper's
order (one chunk + decodes, linears over all rows at once, attention split by token kind with
explicit key ranges [0, q], fp64 KV cache appended in place) — it is what the GPU path must
equal, and the invariant tests prove it equals ``forward_full``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

import synth
from synth import ModelConfig, FFN_SWIGLU, FFN_GELU

# ---------------------------------------------------------------------------
# Weights (bf16 values from the synth generator, upcast exactly to fp64).
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class LayerWeights:
    wq: np.ndarray   # [n_q*hd, H]   (nn.Linear layout [out, in])
    wk: np.ndarray   # [n_kv*hd, H]
    wv: np.ndarray   # [n_kv*hd, H]
    wo: np.ndarray   # [H, n_q*hd]
    wg: np.ndarray   # [H2, H]   (GELU variant: W1)
    wu: Optional[np.ndarray]  # [H2, H]   (None for GELU variant)
    wd: np.ndarray   # [H, H2]   (GELU variant: W2)
    g1: np.ndarray   # [H]
    g2: np.ndarray   # [H]


@dataclasses.dataclass
class ModelWeights:
    cfg: ModelConfig
    emb: np.ndarray      # [V, H]
    layers: List[LayerWeights]
    gf: np.ndarray       # [H]
    wlm: np.ndarray      # [V, H]


def layer_weights(cfg: ModelConfig, seed: int, layer: int) -> LayerWeights:
    f = lambda kind: synth.as_f64(synth.layer_tensor_bits(cfg, seed, layer, kind))
    return LayerWeights(
        wq=f(synth.WQ), wk=f(synth.WK), wv=f(synth.WV), wo=f(synth.WO), wg=f(synth.WG),
        wu=f(synth.WU) if cfg.ffn_kind == FFN_SWIGLU else None, wd=f(synth.WD),
        g1=f(synth.G1), g2=f(synth.G2))


def model_weights(cfg: ModelConfig, seed: int) -> ModelWeights:
    return ModelWeights(
        cfg=cfg,
        emb=synth.as_f64(synth.embedding_bits(cfg, seed)),
        layers=[layer_weights(cfg, seed, l) for l in range(cfg.n_layers)],
        gf=synth.as_f64(synth.final_gain_bits(cfg, seed)),
        wlm=synth.as_f64(synth.lm_head_bits(cfg, seed)))


# ---------------------------------------------------------------------------
# The "others" ops (§2.1: "layer normalization, activation functions, residual").
# ---------------------------------------------------------------------------


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm(x; g) = x / sqrt(mean(x^2) + eps) * g   (reading O-8, eps = 1e-5)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope_tables(pos: np.ndarray, head_dim: int, base: float) -> Tuple[np.ndarray, np.ndarray]:
    """theta_i = base^(-2i/hd), angle = pos * theta_i, i in [0, hd/2)   (reading O-7)."""
    half = head_dim // 2
    inv = base ** (-(np.arange(half, dtype=np.float64) * 2.0) / head_dim)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope(x: np.ndarray, pos: np.ndarray, base: float) -> np.ndarray:
    """Rotate-half RoPE: x [T, n, hd] at positions pos [T]; pairs (i, i + hd/2) (reading O-7)."""
    hd = x.shape[-1]
    half = hd // 2
    cos, sin = rope_tables(pos, hd, base)
    cos, sin = cos[:, None, :], sin[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def kv_head_of(cfg: ModelConfig, q_head: int) -> int:
    """Contiguous GQA grouping kappa(eta) = floor(eta * n_kv / n_q) (reading O-4)."""
    return (q_head * cfg.n_kv_heads) // cfg.n_heads


def ffn(cfg: ModelConfig, w: LayerWeights, b: np.ndarray) -> np.ndarray:
    """ffn_ln1 then ffn_ln2 (Table, shapes [H,H2] and [H2,H])."""
    if cfg.ffn_kind == FFN_SWIGLU:
        return (silu(b @ w.wg.T) * (b @ w.wu.T)) @ w.wd.T
    return gelu_tanh(b @ w.wg.T) @ w.wd.T


# ---------------------------------------------------------------------------
# forward_full: one request, its whole history, dense causal mask, no cache.
# ---------------------------------------------------------------------------


def causal_attention_dense(cfg: ModelConfig, q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """softmax(Q K^T / sqrt(hd) + M) V with M_ij = -inf for j > i (inclusive causal, O-9/O-10).

    q [n, n_q, hd], k/v [n, n_kv, hd] -> o [n, n_q*hd]
    """
    n = q.shape[0]
    hd = cfg.head_dim
    out = np.empty((n, cfg.n_heads, hd))
    mask = np.triu(np.full((n, n), -np.inf), k=1)
    for h in range(cfg.n_heads):
        kh = kv_head_of(cfg, h)
        s = q[:, h, :] @ k[:, kh, :].T / math.sqrt(hd) + mask
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ v[:, kh, :]
    return out.reshape(n, cfg.n_heads * hd)


@dataclasses.dataclass
class FullResult:
    logits: np.ndarray               # [n, V]
    hidden: List[np.ndarray]         # hidden[l] = h^{l+1} [n, H] (residual after layer l)


def forward_full(w: ModelWeights, toks: Sequence[int]) -> FullResult:
    cfg = w.cfg
    toks = np.asarray(toks, dtype=np.int64)
    n = len(toks)
    pos = np.arange(n)
    h = w.emb[toks]
    hidden = []
    for lw in w.layers:
        a = rmsnorm(h, lw.g1, cfg.rms_eps)
        q = rope((a @ lw.wq.T).reshape(n, cfg.n_heads, cfg.head_dim), pos, cfg.rope_base)
        k = rope((a @ lw.wk.T).reshape(n, cfg.n_kv_heads, cfg.head_dim), pos, cfg.rope_base)
        v = (a @ lw.wv.T).reshape(n, cfg.n_kv_heads, cfg.head_dim)
        o = causal_attention_dense(cfg, q, k, v)
        u = h + o @ lw.wo.T
        h = u + ffn(cfg, lw, rmsnorm(u, lw.g2, cfg.rms_eps))
        hidden.append(h.copy())
    logits = rmsnorm(h, w.gf, cfg.rms_eps) @ w.wlm.T
    return FullResult(logits, hidden)


# ---------------------------------------------------------------------------
# Incremental replay of a hybrid-batch schedule (decode-maximal batching, §4.3).
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class PrefillItem:
    req_id: int
    start: int            # s = tokens already cached for the request
    tokens: Sequence[int]  # the chunk's p token ids (positions s .. s+p-1)


@dataclasses.dataclass
class DecodeItem:
    req_id: int
    pos: int              # == cached length of the request (the new token's position)
    token: int


@dataclasses.dataclass
class BatchResult:
    logits: np.ndarray            # [T, V] one row per batch token (chunk rows first, then decodes)
    hidden: List[np.ndarray]      # per layer [T, H]
    positions: np.ndarray         # [T]
    layer_inputs: List[np.ndarray]  # per layer, the residual entering the layer [T, H]


def attention_rows(cfg: ModelConfig, q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray,
                   key_end: int) -> np.ndarray:
    """One query row against keys [0, key_end] inclusive (P:L369 progressive mask; O-9).

    q [n_q, hd]; k_cache/v_cache [>= key_end+1, n_kv, hd] -> [n_q*hd]
    """
    hd = cfg.head_dim
    out = np.empty((cfg.n_heads, hd))
    for h in range(cfg.n_heads):
        kh = kv_head_of(cfg, h)
        s = k_cache[: key_end + 1, kh, :] @ q[h] / math.sqrt(hd)
        s = s - s.max()
        p = np.exp(s)
        out[h] = (p / p.sum()) @ v_cache[: key_end + 1, kh, :]
    return out.reshape(-1)


class IncrementalOracle:
    """Replays hybrid batches with an fp64 per-request KV cache, in the paper's order."""

    def __init__(self, w: ModelWeights):
        self.w = w
        self.cfg = w.cfg
        # kv[req] = list over layers of (K [len, n_kv, hd], V [len, n_kv, hd])
        self.kv: Dict[int, List[Tuple[np.ndarray, np.ndarray]]] = {}

    def cached_len(self, req_id: int) -> int:
        if req_id not in self.kv:
            return 0
        return self.kv[req_id][0][0].shape[0]

    def free(self, req_id: int) -> None:
        self.kv.pop(req_id, None)

    def run_batch(self, prefill: Optional[PrefillItem], decodes: Sequence[DecodeItem]) -> BatchResult:
        cfg, w = self.cfg, self.w
        rows = batch_rows(prefill, decodes, self.cached_len)
        T = len(rows)
        pos = np.array([r[1] for r in rows])
        h = w.emb[np.array([r[2] for r in rows])]           # embedding gather
        hidden, layer_inputs = [], []
        for l, lw in enumerate(w.layers):
            layer_inputs.append(h.copy())
            kv_l = {}
            for rid, _, _ in rows:
                cache = self.kv.setdefault(rid, [(np.zeros((0, cfg.n_kv_heads, cfg.head_dim)),) * 2
                                                 for _ in range(cfg.n_layers)])
                kv_l[rid] = cache[l]
            h = layer_step(cfg, lw, h, rows, kv_l)
            for rid in kv_l:
                self.kv[rid][l] = kv_l[rid]
            hidden.append(h.copy())
        logits = rmsnorm(h, w.gf, cfg.rms_eps) @ w.wlm.T
        return BatchResult(logits, hidden, pos, layer_inputs)


def batch_rows(prefill: Optional[PrefillItem], decodes: Sequence[DecodeItem], cached_len):
    """Token matrix of one hybrid batch (§4.3): the chunk's rows (positions s..s+p-1) then one row
    per decode (position = its cached length); (req, pos, token) per row."""
    rows: List[Tuple[int, int, int]] = []
    if prefill is not None:
        assert prefill.start == cached_len(prefill.req_id), "chunk must start at cached length"
        for i, t in enumerate(prefill.tokens):
            rows.append((prefill.req_id, prefill.start + i, int(t)))
    seen = {prefill.req_id} if prefill is not None else set()
    for d in decodes:
        assert d.req_id not in seen, "a request appears once per batch (S:L443)"
        seen.add(d.req_id)
        assert d.pos == cached_len(d.req_id) and d.pos > 0, "decode at cached length"
        rows.append((d.req_id, d.pos, int(d.token)))
    assert len(rows) > 0
    return rows


def layer_step(cfg: ModelConfig, lw: LayerWeights, h: np.ndarray, rows, kv_l) -> np.ndarray:
    """One decoder layer over the batch's rows, in the paper's order: linears over all T rows at once
    ("fuse all the linear operations"), K/V appended in place to each request's cache of this
    layer (kv_l[req] = (K, V), replaced by the extended arrays), attention split by
    token kind with explicit key ranges [0, pos] (P:L369 progressive mask; reading O-9)."""
    T = h.shape[0]
    pos = np.array([r[1] for r in rows])
    a = rmsnorm(h, lw.g1, cfg.rms_eps)
    q = rope((a @ lw.wq.T).reshape(T, cfg.n_heads, cfg.head_dim), pos, cfg.rope_base)
    k = rope((a @ lw.wk.T).reshape(T, cfg.n_kv_heads, cfg.head_dim), pos, cfg.rope_base)
    v = (a @ lw.wv.T).reshape(T, cfg.n_kv_heads, cfg.head_dim)
    # KV-cache in-place append (P:L112 pre-allocated cache).
    for i, (rid, p_, _) in enumerate(rows):
        K, V = kv_l[rid]
        assert K.shape[0] == p_
        kv_l[rid] = (np.concatenate([K, k[i:i + 1]]), np.concatenate([V, v[i:i + 1]]))
    # Attention split by token kind: prefill rows attend [0, s+i], decodes [0, ctx-1].
    o = np.empty((T, cfg.q_dim))
    for i, (rid, p_, _) in enumerate(rows):
        K, V = kv_l[rid]
        o[i] = attention_rows(cfg, q[i], K, V, p_)
    u = h + o @ lw.wo.T
    return u + ffn(cfg, lw, rmsnorm(u, lw.g2, cfg.rms_eps))


def replay_layer_major(cfg: ModelConfig, layer_weights_fn, emb_rows_fn, gf: np.ndarray, wlm: np.ndarray,
                       batches) -> List[BatchResult]:
    """The same computation as IncrementalOracle.run_batch over a sequence of batches, reordered
    layer-major: every batch through layer 0, then every batch through layer 1, ...  Exact (each
    batch's layer-l input and each request's layer-l KV are the same arrays in either order), so a
    full-size model (e.g. 40 LLaMA-13B layers) needs ONE layer's fp64 weights in memory at a time.
    layer_weights_fn(l) -> LayerWeights; emb_rows_fn(token ids) -> fp64 embedding rows;
    batches = [(PrefillItem | None, [DecodeItem])]."""
    lens: Dict[int, int] = {}
    rows_b = []
    for pre, decs in batches:
        rows = batch_rows(pre, decs, lambda r: lens.get(r, 0))
        for rid, _, _ in rows:
            lens[rid] = lens.get(rid, 0) + 1
        rows_b.append(rows)
    h_b = [emb_rows_fn(np.array([r[2] for r in rows])) for rows in rows_b]
    hidden_b: List[List[np.ndarray]] = [[] for _ in rows_b]
    inputs_b: List[List[np.ndarray]] = [[] for _ in rows_b]
    for l in range(cfg.n_layers):
        lw = layer_weights_fn(l)
        kv_l: Dict[int, Tuple[np.ndarray, np.ndarray]] = {}
        for b, rows in enumerate(rows_b):
            for rid, _, _ in rows:
                kv_l.setdefault(rid, (np.zeros((0, cfg.n_kv_heads, cfg.head_dim)),) * 2)
            inputs_b[b].append(h_b[b].copy())
            h_b[b] = layer_step(cfg, lw, h_b[b], rows, kv_l)
            hidden_b[b].append(h_b[b].copy())
        del lw
    out = []
    for b, rows in enumerate(rows_b):
        logits = rmsnorm(h_b[b], gf, cfg.rms_eps) @ wlm.T
        out.append(BatchResult(logits, hidden_b[b], np.array([r[1] for r in rows]), inputs_b[b]))
    return out


# ---------------------------------------------------------------------------
# Layer-local evaluation (SURVEY §8(c) compare mode "layer-local") for full-size checks.
# ---------------------------------------------------------------------------


def layer_rows_from_input(cfg: ModelConfig, lw: LayerWeights, h_in: np.ndarray, pos: np.ndarray,
                          k_ctx: Sequence[np.ndarray], v_ctx: Sequence[np.ndarray]) -> np.ndarray:
    """One layer for a few rows given their residual input and the KV each row attends.

    h_in [n, H]; pos [n]; k_ctx[i]/v_ctx[i] = [pos_i+1, n_kv, hd] keys/values of the row's
    request for positions [0, pos_i] (the row's own post-RoPE k / v included as the last entry).
    Returns h_out [n, H].
    """
    n = h_in.shape[0]
    a = rmsnorm(h_in, lw.g1, cfg.rms_eps)
    q = rope((a @ lw.wq.T).reshape(n, cfg.n_heads, cfg.head_dim), pos, cfg.rope_base)
    o = np.stack([attention_rows(cfg, q[i], k_ctx[i], v_ctx[i], int(pos[i])) for i in range(n)])
    u = h_in + o @ lw.wo.T
    return u + ffn(cfg, lw, rmsnorm(u, lw.g2, cfg.rms_eps))


def qkv_rows(cfg: ModelConfig, lw: LayerWeights, h_in: np.ndarray, pos: np.ndarray):
    """Post-RoPE q, k and v of rows (used to check the fused KV append at full size)."""
    n = h_in.shape[0]
    a = rmsnorm(h_in, lw.g1, cfg.rms_eps)
    q = rope((a @ lw.wq.T).reshape(n, cfg.n_heads, cfg.head_dim), pos, cfg.rope_base)
    k = rope((a @ lw.wk.T).reshape(n, cfg.n_kv_heads, cfg.head_dim), pos, cfg.rope_base)
    v = (a @ lw.wv.T).reshape(n, cfg.n_kv_heads, cfg.head_dim)
    return q, k, v


def logits_rows(cfg: ModelConfig, gf: np.ndarray, wlm_rows: np.ndarray, h_final: np.ndarray) -> np.ndarray:
    """Final norm + LM head restricted to a subset of vocab rows: [n, len(wlm_rows)]."""
    return rmsnorm(h_final, gf, cfg.rms_eps) @ wlm_rows.T

"""Pins for oracle/model.py against things other than itself:
library (HF LlamaForCausalLM in float64, torch activations), closed forms, scalar-loop brute
force, and the method's exact invariants (P:L369 chunked == full; P:L403 hybrid == alone;
P:L224 cached decode == recomputation)."""
import dataclasses
import math

import numpy as np
import pytest
import torch

import synth
from oracle import model as om
from oracle import sched as osch

TINY_GQA = dataclasses.replace(synth.TINY, name="tiny-gqa", n_kv_heads=2)
MICRO = synth.ModelConfig("micro", 1, 8, 2, 1, 4, 16, 16, max_seq_len=16)


@pytest.fixture(scope="module")
def tiny_w():
    return om.model_weights(synth.TINY, 0)


@pytest.fixture(scope="module")
def gqa_w():
    return om.model_weights(TINY_GQA, 7)


# ---------------------------------------------------------------------------
# Library pin: HF LlamaForCausalLM (float64) loaded with the same weights.
# ---------------------------------------------------------------------------

def _hf_model(w: om.ModelWeights, exact_rope: bool):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = w.cfg
    hc = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn_hidden,
                     num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                     num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                     max_position_embeddings=cfg.max_seq_len, rms_norm_eps=cfg.rms_eps,
                     rope_theta=cfg.rope_base, tie_word_embeddings=False, attention_bias=False,
                     mlp_bias=False, attn_implementation="sdpa")
    m = LlamaForCausalLM(hc).to(torch.float64).eval()
    sd = {"model.embed_tokens.weight": w.emb, "model.norm.weight": w.gf, "lm_head.weight": w.wlm}
    for l, lw in enumerate(w.layers):
        p = f"model.layers.{l}."
        sd.update({p + "self_attn.q_proj.weight": lw.wq, p + "self_attn.k_proj.weight": lw.wk,
                   p + "self_attn.v_proj.weight": lw.wv, p + "self_attn.o_proj.weight": lw.wo,
                   p + "mlp.gate_proj.weight": lw.wg, p + "mlp.up_proj.weight": lw.wu,
                   p + "mlp.down_proj.weight": lw.wd, p + "input_layernorm.weight": lw.g1,
                   p + "post_attention_layernorm.weight": lw.g2})
    m.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()}, strict=False)
    if exact_rope:
        # HF computes the RoPE angles in float32; recompute them in float64 (textbook
        # theta_i = base^(-2i/d)) so the comparison can be held to 1e-10.
        rot = m.model.rotary_emb
        d = cfg.head_dim

        def fwd(x, position_ids):
            inv = 1.0 / (cfg.rope_base ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
            fr = position_ids.to(torch.float64)[..., None] * inv
            emb = torch.cat([fr, fr], dim=-1)
            return emb.cos().to(x.dtype), emb.sin().to(x.dtype)
        rot.forward = fwd
        # HF's LlamaRMSNorm also upcasts to float32 internally; keep it in float64.
        from transformers.models.llama.modeling_llama import LlamaRMSNorm
        for mod in m.modules():
            if isinstance(mod, LlamaRMSNorm):
                def nf(x, mod=mod):
                    var = x.pow(2).mean(-1, keepdim=True)
                    return mod.weight * (x * torch.rsqrt(var + mod.variance_epsilon))
                mod.forward = nf
    return m


@pytest.mark.parametrize("which", ["tiny", "gqa"])
@pytest.mark.parametrize("exact_rope", [True, False])
def test_forward_full_matches_hf_llama_fp64(which, exact_rope, tiny_w, gqa_w):
    w = tiny_w if which == "tiny" else gqa_w
    toks = synth.tokens(3, 1, 0, 48, w.cfg.vocab)
    ours = om.forward_full(w, toks)
    m = _hf_model(w, exact_rope)
    with torch.no_grad():
        out = m(torch.from_numpy(toks.astype(np.int64))[None], output_hidden_states=True)
    ref = out.logits[0].numpy()
    tol = 1e-10 if exact_rope else 2e-5
    rel = np.max(np.abs(ours.logits - ref)) / np.max(np.abs(ref))
    assert rel < tol, rel
    # residual after every layer but the last (HF replaces the last with the normed state)
    for l in range(w.cfg.n_layers - 1):
        hr = out.hidden_states[l + 1][0].numpy()
        assert np.max(np.abs(ours.hidden[l] - hr)) / np.max(np.abs(hr)) < tol


# ---------------------------------------------------------------------------
# Closed forms and special cases.
# ---------------------------------------------------------------------------

def test_rmsnorm_closed_form_and_invariances():
    x = np.array([[3.0, 4.0]])
    g = np.array([1.0, 2.0])
    r = math.sqrt((9 + 16) / 2)
    assert np.allclose(om.rmsnorm(x, g, 0.0), [[3 / r, 8 / r]], rtol=0, atol=1e-15)
    rng = np.random.default_rng(1)
    v = rng.standard_normal((4, 64))
    gg = rng.standard_normal(64)
    assert np.allclose(om.rmsnorm(7.5 * v, gg, 0.0), om.rmsnorm(v, gg, 0.0), atol=1e-13)
    c = np.full((1, 64), -2.0)
    assert np.allclose(om.rmsnorm(c, gg, 0.0), -gg[None])
    # eps enters as mean(x^2) + eps: for x = 0 the result is 0, for tiny x it damps
    assert np.allclose(om.rmsnorm(np.zeros((1, 4)), np.ones(4), 1e-5), 0.0)


def test_rope_identity_at_zero_and_norm_preserving():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((5, 3, 64))
    assert np.allclose(om.rope(x, np.zeros(5), 10000.0), x, atol=0)
    y = om.rope(x, np.arange(5) * 37, 10000.0)
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), atol=1e-12)


def test_rope_equals_complex_rotation():
    rng = np.random.default_rng(3)
    hd, half = 64, 32
    x = rng.standard_normal((6, 1, hd))
    pos = np.array([0, 1, 5, 100, 1023, 4095])
    y = om.rope(x, pos, 10000.0)
    z = x[..., :half] + 1j * x[..., half:]
    theta = 10000.0 ** (-np.arange(half) * 2.0 / hd)
    zr = z * np.exp(1j * pos[:, None, None] * theta[None, None, :])
    assert np.allclose(y[..., :half], zr.real, atol=1e-12)
    assert np.allclose(y[..., half:], zr.imag, atol=1e-12)


def test_rope_relative_position_property():
    rng = np.random.default_rng(4)
    q = rng.standard_normal((1, 1, 64))
    k = rng.standard_normal((1, 1, 64))
    dots = []
    for m, n in [(10, 3), (107, 100), (2007, 2000)]:
        a = om.rope(q, np.array([m]), 10000.0)
        b = om.rope(k, np.array([n]), 10000.0)
        dots.append(float((a * b).sum()))
    assert np.allclose(dots, dots[0], atol=1e-10)


def test_activations_match_torch():
    x = np.linspace(-12, 12, 2001)
    tx = torch.from_numpy(x)
    assert np.allclose(om.silu(x), torch.nn.functional.silu(tx).numpy(), atol=1e-15)
    assert np.allclose(om.gelu_tanh(x), torch.nn.functional.gelu(tx, approximate="tanh").numpy(), atol=1e-15)
    assert om.silu(np.array([0.0]))[0] == 0.0
    assert abs(om.silu(np.array([40.0]))[0] - 40.0) < 1e-12


def test_attention_zero_query_is_running_mean():
    cfg = synth.TINY
    rng = np.random.default_rng(5)
    n = 9
    q = np.zeros((n, cfg.n_heads, cfg.head_dim))
    k = rng.standard_normal((n, cfg.n_kv_heads, cfg.head_dim))
    v = rng.standard_normal((n, cfg.n_kv_heads, cfg.head_dim))
    o = om.causal_attention_dense(cfg, q, k, v).reshape(n, cfg.n_heads, cfg.head_dim)
    mean = np.cumsum(v, axis=0) / np.arange(1, n + 1)[:, None, None]
    assert np.allclose(o, mean, atol=1e-14)
    for i in range(n):
        r = om.attention_rows(cfg, q[i], k, v, i).reshape(cfg.n_heads, cfg.head_dim)
        assert np.allclose(r, mean[i], atol=1e-14)


def test_attention_single_key_and_duplicate_keys():
    cfg = TINY_GQA
    rng = np.random.default_rng(6)
    q = rng.standard_normal((cfg.n_heads, cfg.head_dim))
    k = rng.standard_normal((1, cfg.n_kv_heads, cfg.head_dim))
    v = rng.standard_normal((1, cfg.n_kv_heads, cfg.head_dim))
    o = om.attention_rows(cfg, q, k, v, 0).reshape(cfg.n_heads, cfg.head_dim)
    for h in range(cfg.n_heads):
        assert np.allclose(o[h], v[0, om.kv_head_of(cfg, h)])
    k2, v2 = np.concatenate([k, k]), np.concatenate([v, v])
    assert np.allclose(om.attention_rows(cfg, q, k2, v2, 1), o.reshape(-1), atol=1e-15)


def test_gqa_grouping_contiguous():
    cfg = synth.LLAMA2_70B
    assert [om.kv_head_of(cfg, h) for h in (0, 7, 8, 63)] == [0, 0, 1, 7]


def test_dense_mask_equals_key_range_loop():
    cfg = TINY_GQA
    rng = np.random.default_rng(7)
    n = 13
    q = rng.standard_normal((n, cfg.n_heads, cfg.head_dim))
    k = rng.standard_normal((n, cfg.n_kv_heads, cfg.head_dim))
    v = rng.standard_normal((n, cfg.n_kv_heads, cfg.head_dim))
    dense = om.causal_attention_dense(cfg, q, k, v)
    loop = np.stack([om.attention_rows(cfg, q[i], k, v, i) for i in range(n)])
    assert np.max(np.abs(dense - loop)) < 1e-13


# ---------------------------------------------------------------------------
# Scalar-loop brute force of one whole forward at H = 8 (pure Python, no NumPy algebra).
# ---------------------------------------------------------------------------

def _scalar_forward(w: om.ModelWeights, toks, trace=None):
    """Pure-Python loops; `trace` (optional dict) receives per layer l the residual entering the
    layer ("h_in", l) and the post-RoPE q / k and v of every token ("q"/"k"/"v", l)."""
    cfg = w.cfg
    H, hd, nq, nkv = cfg.hidden, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    W = lambda a: a.tolist()

    def mv(mat, x):
        return [sum(mat[r][c] * x[c] for c in range(len(x))) for r in range(len(mat))]

    def norm(x, g):
        ms = sum(t * t for t in x) / len(x)
        return [x[i] / math.sqrt(ms + cfg.rms_eps) * g[i] for i in range(len(x))]

    def rot(vec, p):
        out = list(vec)
        half = hd // 2
        for i in range(half):
            th = p * cfg.rope_base ** (-2.0 * i / hd)
            a, b = vec[i], vec[i + half]
            out[i] = a * math.cos(th) - b * math.sin(th)
            out[i + half] = b * math.cos(th) + a * math.sin(th)
        return out

    gelu = cfg.ffn_kind == synth.FFN_GELU
    hs = [W(w.emb[t]) for t in toks]
    for l, lw in enumerate(w.layers):
        wq, wk, wv, wo, wg, wd = map(W, (lw.wq, lw.wk, lw.wv, lw.wo, lw.wg, lw.wd))
        wu = None if gelu else W(lw.wu)
        Ks, Vs, new, Qs = [], [], [], []
        if trace is not None:
            trace[("h_in", l)] = [list(h) for h in hs]
        for i, h in enumerate(hs):
            a = norm(h, W(lw.g1))
            q, k, v = mv(wq, a), mv(wk, a), mv(wv, a)
            qh = [rot(q[j * hd:(j + 1) * hd], i) for j in range(nq)]
            Ks.append([rot(k[j * hd:(j + 1) * hd], i) for j in range(nkv)])
            Vs.append([v[j * hd:(j + 1) * hd] for j in range(nkv)])
            Qs.append(qh)
            o = []
            for j in range(nq):
                kv = j * nkv // nq
                sc = [sum(qh[j][c] * Ks[t][kv][c] for c in range(hd)) / math.sqrt(hd) for t in range(i + 1)]
                mx = max(sc)
                e = [math.exp(s - mx) for s in sc]
                z = sum(e)
                o += [sum(e[t] / z * Vs[t][kv][c] for t in range(i + 1)) for c in range(hd)]
            u = [h[c] + x for c, x in enumerate(mv(wo, o))]
            b = norm(u, W(lw.g2))
            if gelu:  # ffn_ln1 -> GELU-tanh -> ffn_ln2 (Table; reading O-1)
                z = mv(wg, b)
                f = [0.5 * x * (1 + math.tanh(math.sqrt(2 / math.pi) * (x + 0.044715 * x * x * x))) for x in z]
            else:
                gate, up = mv(wg, b), mv(wu, b)
                f = [gate[r] / (1 + math.exp(-gate[r])) * up[r] for r in range(len(gate))]
            new.append([u[c] + x for c, x in enumerate(mv(wd, f))])
        if trace is not None:
            trace[("q", l)], trace[("k", l)], trace[("v", l)] = Qs, Ks, Vs
        hs = new
    wlm = W(w.wlm)
    return [mv(wlm, norm(h, W(w.gf))) for h in hs]


MICRO_GELU = dataclasses.replace(MICRO, name="micro-gelu", n_layers=2, ffn_kind=synth.FFN_GELU, ffn_hidden=32)


@pytest.mark.parametrize("cfg", [MICRO, MICRO_GELU], ids=["swiglu", "gelu"])
def test_forward_full_matches_scalar_loops(cfg):
    """Whole forward vs pure-Python loops; the GELU case pins the 2-matrix ffn branch
    (GELU-tanh after W1, then W2; Table), which has no HF twin."""
    w = om.model_weights(cfg, 9)
    toks = [3, 15, 0, 3, 7]
    ref = np.array(_scalar_forward(w, toks))
    ours = om.forward_full(w, toks).logits
    assert np.max(np.abs(ours - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_gelu_ffn_branch_order():
    """ffn() GELU branch = W2 . GELU(W1 b): applying GELU after W2 instead (a plausible slip)
    or using SiLU gives a different answer, so the scalar-loop pin above really covers it."""
    w = om.model_weights(MICRO_GELU, 4)
    lw = w.layers[0]
    b = np.random.default_rng(0).standard_normal((3, MICRO_GELU.hidden))
    got = om.ffn(MICRO_GELU, lw, b)
    z = b @ lw.wg.T
    ref = np.array([[sum(0.5 * x * (1 + math.tanh(math.sqrt(2 / math.pi) * (x + 0.044715 * x ** 3))) * lw.wd[c, r]
                         for r, x in enumerate(row)) for c in range(MICRO_GELU.hidden)] for row in z])
    assert np.max(np.abs(got - ref)) < 1e-12
    assert np.max(np.abs(om.gelu_tanh(z @ lw.wd.T) - ref)) > 1e-3


def test_qkv_rows_matches_scalar_loops():
    """Post-RoPE q, k and v of qkv_rows (the full-size KV-append checker) vs the scalar loops'
    per-token q/k/v at every position (RoPE at the row's own position, P:L214 fused QKV)."""
    for cfg in (MICRO, MICRO_GELU):
        w = om.model_weights(cfg, 9)
        toks = [3, 15, 0, 3, 7, 11]
        tr = {}
        _scalar_forward(w, toks, tr)
        for l in range(cfg.n_layers):
            h_in = np.array(tr[("h_in", l)])
            pos = np.arange(len(toks))
            q, k, v = om.qkv_rows(cfg, w.layers[l], h_in, pos)
            assert np.max(np.abs(q - np.array(tr[("q", l)]))) < 1e-12
            assert np.max(np.abs(k - np.array(tr[("k", l)]))) < 1e-12
            assert np.max(np.abs(v - np.array(tr[("v", l)]))) < 1e-12
            # a subset of rows at their own positions gives the same rows (no dependence on batch)
            sel = np.array([5, 1])
            q2, k2, _ = om.qkv_rows(cfg, w.layers[l], h_in[sel], pos[sel])
            assert np.max(np.abs(q2 - q[sel])) < 1e-12 and np.max(np.abs(k2 - k[sel])) < 1e-12


@pytest.mark.parametrize("which", ["tiny", "gqa"])
def test_layer_local_helpers_equal_incremental_replay(which, tiny_w, gqa_w):
    """layer_rows_from_input / qkv_rows / logits_rows (the checkers behind the full-size GPU
    parity tests) equal the incremental replay's per-layer rows, appended K/V and logits for
    chunk rows and decode rows, including positions at 16- and 64-token block boundaries."""
    w = tiny_w if which == "tiny" else gqa_w
    cfg = w.cfg
    V = cfg.vocab
    toks = {r: synth.tokens(23, r, 0, 80, V) for r in (0, 1, 2)}
    o = om.IncrementalOracle(w)
    o.run_batch(om.PrefillItem(1, 0, toks[1][:16]), [])          # request 1 cached [0, 16)
    o.run_batch(om.PrefillItem(2, 0, toks[2][:63]), [])          # request 2 cached [0, 63)
    o.run_batch(om.PrefillItem(0, 0, toks[0][:15]), [])
    # hybrid batch: chunk of request 0 at s = 15 (rows at positions 15, 16, ... 31, 32) + decodes
    # of request 1 at position 16 and request 2 at 63 (block boundaries for bs 16 / 64)
    res = o.run_batch(om.PrefillItem(0, 15, toks[0][15:33]),
                      [om.DecodeItem(1, 16, toks[1][16]), om.DecodeItem(2, 63, toks[2][63])])
    p = 18
    rows = [0, 1, p - 1, p, p + 1]
    req = [0, 0, 0, 1, 2]
    pos = np.array([15, 16, 32, 16, 63])
    assert np.array_equal(res.positions[rows], pos)
    for l in range(cfg.n_layers):
        h_in = res.layer_inputs[l][rows]
        kctx = [o.kv[r][l][0][:ps + 1] for r, ps in zip(req, pos)]
        vctx = [o.kv[r][l][1][:ps + 1] for r, ps in zip(req, pos)]
        got = om.layer_rows_from_input(cfg, w.layers[l], h_in, pos, kctx, vctx)
        assert _rel(got, res.hidden[l][rows]) < 1e-12, l
        _, k, v = om.qkv_rows(cfg, w.layers[l], h_in, pos)
        assert np.max(np.abs(k - np.stack([kc[-1] for kc in kctx]))) < 1e-12
        assert np.max(np.abs(v - np.stack([vc[-1] for vc in vctx]))) < 1e-12
        # dropping the row's own key (key_end = pos - 1, reading O-9 violated) is detected
        short = [kc[:-1] for kc in kctx]
        bad = om.layer_rows_from_input(cfg, w.layers[l], h_in[1:], pos[1:] - 1, short[1:], [vc[:-1] for vc in vctx][1:])
        assert _rel(bad, res.hidden[l][rows[1:]]) > 1e-6
    vidx = np.arange(3, V, 7)
    lg = om.logits_rows(cfg, w.gf, w.wlm[vidx], res.hidden[-1][rows])
    assert _rel(lg, res.logits[rows][:, vidx]) < 1e-12


def test_relative_error_hand_example():
    """||gpu - ref||_inf / ||ref||_inf (reading O-20) on hand-computed values."""
    from oracle.metrics import relative_error
    assert relative_error([1.0, 2.5, -3.0], [1.0, 2.0, -4.0]) == pytest.approx(0.25, abs=0)
    assert relative_error([[0.5, -1.0]], [[0.0, 0.0]]) == 1.0       # zero reference: absolute error
    assert relative_error(np.float32([2.0]), np.float64([2.0])) == 0.0
    assert relative_error([-8.0, 1.0], [-10.0, 0.0]) == pytest.approx(0.2)   # sign-aware, inf-norm of ref


# ---------------------------------------------------------------------------
# The method's invariants, exact in R, asserted at 1e-12 relative in fp64.
# ---------------------------------------------------------------------------

def _rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def test_chunked_prefill_equals_full_for_every_chunk_size(tiny_w):
    P = 20
    toks = synth.tokens(5, 0, 0, P, tiny_w.cfg.vocab)
    full = om.forward_full(tiny_w, toks)
    for C in range(1, P + 1):
        o = om.IncrementalOracle(tiny_w)
        rows = []
        for s, n in osch.plan_chunks(P, C):
            r = o.run_batch(om.PrefillItem(0, s, toks[s:s + n]), [])
            rows.append(r.logits)
        got = np.concatenate(rows)
        assert _rel(got, full.logits) < 1e-12, C
        # final KV store equals the one a single full-prefill pass would build
        o2 = om.IncrementalOracle(tiny_w)
        o2.run_batch(om.PrefillItem(0, 0, toks), [])
        for l in range(tiny_w.cfg.n_layers):
            assert np.max(np.abs(o.kv[0][l][0] - o2.kv[0][l][0])) < 1e-12


def test_hybrid_batch_equals_each_request_alone_and_decode_equals_recompute(gqa_w):
    cfg = gqa_w.cfg
    V = cfg.vocab
    # Requests: A prefilled in chunks of 6 while B and C decode alongside (decode-maximal batch).
    toks = {r: synth.tokens(17, r, 0, 40, V) for r in (0, 1, 2)}
    o = om.IncrementalOracle(gqa_w)
    got = {0: {}, 1: {}, 2: {}}
    o.run_batch(om.PrefillItem(1, 0, toks[1][:9]), [])
    o.run_batch(om.PrefillItem(2, 0, toks[2][:4]), [om.DecodeItem(1, 9, toks[1][9])])
    pos = {1: 10, 2: 4}
    for s, n in osch.plan_chunks(23, 6):
        decs = [om.DecodeItem(r, pos[r], toks[r][pos[r]]) for r in (1, 2)]
        res = o.run_batch(om.PrefillItem(0, s, toks[0][s:s + n]), decs)
        for i in range(n):
            got[0][s + i] = res.logits[i]
        for j, r in enumerate((1, 2)):
            got[r][pos[r]] = res.logits[n + j]
            pos[r] += 1
    for r in (0, 1, 2):
        last = max(got[r])
        full = om.forward_full(gqa_w, toks[r][:last + 1]).logits
        for p_, row in got[r].items():
            assert _rel(row, full[p_]) < 1e-12, (r, p_)


@pytest.mark.parametrize("which", ["tiny", "gqa"])
def test_layer_major_replay_equals_incremental(which, tiny_w, gqa_w):
    """replay_layer_major (the full-size end-to-end checker: one layer's weights in memory at a time)
    reorders IncrementalOracle's work layer-major; the results are the same arrays (bitwise), for a
    schedule with chunks, piggybacked decodes and decode-only batches."""
    w = tiny_w if which == "tiny" else gqa_w
    V = w.cfg.vocab
    toks = {r: synth.tokens(31, r, 0, 60, V) for r in (0, 1, 2)}
    batches = [(om.PrefillItem(1, 0, toks[1][:7]), []),
               (om.PrefillItem(0, 0, toks[0][:16]), [om.DecodeItem(1, 7, toks[1][7])]),
               (om.PrefillItem(0, 16, toks[0][16:21]), [om.DecodeItem(1, 8, toks[1][8])]),
               (om.PrefillItem(2, 0, toks[2][:3]), [om.DecodeItem(0, 21, toks[0][21]), om.DecodeItem(1, 9, toks[1][9])]),
               (None, [om.DecodeItem(2, 3, toks[2][3]), om.DecodeItem(0, 22, toks[0][22])])]
    o = om.IncrementalOracle(w)
    ref = [o.run_batch(p, d) for p, d in batches]
    got = om.replay_layer_major(w.cfg, lambda l: w.layers[l], lambda t: w.emb[t], w.gf, w.wlm, batches)
    for a, b in zip(got, ref):
        assert np.array_equal(a.logits, b.logits)
        assert np.array_equal(a.positions, b.positions)
        for x, y in zip(a.hidden, b.hidden):
            assert np.array_equal(x, y)

"""Shared driver for GPU parity tests: runs a request schedule through the C ABI (C++ scheduler
-> run_hybrid_batch) and, step by step, through the fp64 oracle replay.  Test-only code."""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

import numpy as np

import synth
from oracle import model as om
from oracle import sched as osch
from oracle.metrics import relative_error


@dataclasses.dataclass
class StepResult:
    plan: tuple
    gpu_logits: np.ndarray
    ref_logits: np.ndarray
    gpu_hidden: List[np.ndarray]
    ref_hidden: List[np.ndarray]
    gpu_slots: np.ndarray
    ref_slots: np.ndarray


def run_schedule(S, cfg: synth.ModelConfig, reqs: Sequence[Tuple[int, int, int, int]], B: int, C: int,
                 num_blocks: int, block_size: int, weight_seed: int = 0, tok_seed: int = 1001,
                 max_tokens: int = 64, dump: bool = True, oracle_weights=None,
                 host_tensors=None) -> List[StepResult]:
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=max_tokens), seed=weight_seed, host_tensors=host_tensors)
    m.alloc_kv(num_blocks, block_size)
    sched = S.Scheduler(B, C, num_blocks, block_size)
    for r in reqs:
        sched.submit(*r)
    info = {r[0]: (r[1], r[2]) for r in reqs}
    w = oracle_weights if oracle_weights is not None else om.model_weights(cfg, weight_seed)
    orc = om.IncrementalOracle(w)
    palloc = osch.BlockAllocator(num_blocks, block_size)
    V = cfg.vocab
    tok = lambda rid, pos, n=1: synth.tokens(tok_seed, rid, pos, n, V)
    out = []
    while not sched.done():
        plan, admitted = sched.next()
        for rid in admitted:
            P, D = info[rid]
            m.request_alloc(rid, P + D)
            palloc.alloc(rid, P + D)
        if plan is None:
            sched.idle_step()
            continue
        pre, decs = plan
        prefill = None
        opre = None
        ref_slots = []
        if pre is not None:
            rid, start, n = pre
            t = tok(rid, start, n)
            prefill = (rid, start, t)
            opre = om.PrefillItem(rid, start, t)
            ref_slots += [palloc.slot(rid, start + i) for i in range(n)]
        decodes, odec = [], []
        for rid, pos in decs:
            t = int(tok(rid, pos)[0])
            decodes.append((rid, t, pos))
            odec.append(om.DecodeItem(rid, pos, t))
            ref_slots.append(palloc.slot(rid, pos))
        T = (pre[2] if pre else 0) + len(decs)
        logits = np.zeros((T, V), dtype=np.float32)
        flags = S.RETURN_ALL_ROWS | (S.DUMP_LAYERS if dump else 0)
        m.run_hybrid_batch(prefill, decodes, flags=flags, logits_host=logits)
        hid = [m.hidden(l, T) for l in range(cfg.n_layers)] if dump else []
        ref = orc.run_batch(opre, odec)
        out.append(StepResult(plan, logits, ref.logits, hid, ref.hidden, m.slot_mapping(), np.array(ref_slots)))
        for rid in sched.complete():
            m.request_free(rid)
            palloc.free(rid)
            orc.free(rid)
    m.close()
    return out


def synth_host_tensors(cfg: synth.ModelConfig, seed: int):
    """The logical bf16 weights (uint16 bits) in sarathi_init_model's host_tensors order, produced
    by the synth generator on the host (the seed path generates the same bits on device)."""
    out = []
    for l in range(cfg.n_layers):
        for k in (synth.WQ, synth.WK, synth.WV, synth.WO, synth.WG, synth.WU, synth.WD, synth.G1, synth.G2):
            out.append(None if (k == synth.WU and cfg.ffn_kind == synth.FFN_GELU)
                       else synth.layer_tensor_bits(cfg, seed, l, k))
    out += [synth.embedding_bits(cfg, seed), synth.final_gain_bits(cfg, seed), synth.lm_head_bits(cfg, seed)]
    return out


def worst_errors(steps: Sequence[StepResult]) -> Dict[str, float]:
    e = {"logits": 0.0, "hidden": 0.0}
    for s in steps:
        e["logits"] = max(e["logits"], relative_error(s.gpu_logits, s.ref_logits))
        for g, r in zip(s.gpu_hidden, s.ref_hidden):
            e["hidden"] = max(e["hidden"], relative_error(g, r))
    return e

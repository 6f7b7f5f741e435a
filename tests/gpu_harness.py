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


def gpu_schedule(S, m, cfg: synth.ModelConfig, reqs: Sequence[Tuple[int, int, int, int]], B: int, C: int,
                 num_blocks: int, block_size: int, tok_seed: int = 1001, dump: bool = True):
    """Drives one model handle through the C++ scheduler; returns per step (plan, prefill, decodes,
    logits, hidden, slots).  Under a local TP group every rank's thread calls this identically."""
    sched = S.Scheduler(B, C, num_blocks, block_size)
    for r in reqs:
        sched.submit(*r)
    info = {r[0]: (r[1], r[2]) for r in reqs}
    V = cfg.vocab
    tok = lambda rid, pos, n=1: synth.tokens(tok_seed, rid, pos, n, V)
    out = []
    pending_adm = []  # admitted on idle iterations: replayed before the next step
    while not sched.done():
        plan, admitted = sched.next()
        for rid in admitted:
            P, D = info[rid]
            m.request_alloc(rid, P + D)
        pending_adm += admitted
        if plan is None:
            sched.idle_step()
            continue
        pre, decs = plan
        prefill = None
        if pre is not None:
            rid, start, n = pre
            prefill = (rid, start, tok(rid, start, n))
        decodes = [(rid, int(tok(rid, pos)[0]), pos) for rid, pos in decs]
        T = (pre[2] if pre else 0) + len(decs)
        logits = np.zeros((T, V), dtype=np.float32)
        flags = S.RETURN_ALL_ROWS | (S.DUMP_LAYERS if dump else 0)
        m.run_hybrid_batch(prefill, decodes, flags=flags, logits_host=logits)
        hid = [m.hidden(l, T) for l in range(cfg.n_layers)] if dump else []
        fin = sched.complete()
        out.append(dict(plan=plan, prefill=prefill, decodes=decodes, logits=logits, hidden=hid,
                        slots=m.slot_mapping(), admitted=pending_adm, finished=fin))
        pending_adm = []
        for rid in fin:
            m.request_free(rid)
    return out, info


def oracle_schedule(w, gpu_steps, info, num_blocks: int, block_size: int) -> List[StepResult]:
    """Replays the same batches through the fp64 incremental oracle and the Python allocator."""
    orc = om.IncrementalOracle(w)
    palloc = osch.BlockAllocator(num_blocks, block_size)
    out = []
    for st in gpu_steps:
        for rid in st["admitted"]:  # same admission order as the library's allocator
            P, D = info[rid]
            palloc.alloc(rid, P + D)
        opre = None
        ref_slots = []
        if st["prefill"] is not None:
            rid, start, t = st["prefill"]
            opre = om.PrefillItem(rid, start, t)
            ref_slots += [palloc.slot(rid, start + i) for i in range(len(t))]
        odec = []
        for rid, t, pos in st["decodes"]:
            odec.append(om.DecodeItem(rid, pos, t))
            ref_slots.append(palloc.slot(rid, pos))
        ref = orc.run_batch(opre, odec)
        out.append(StepResult(st["plan"], st["logits"], ref.logits, st["hidden"], ref.hidden, st["slots"],
                              np.array(ref_slots)))
        for rid in st["finished"]:
            palloc.free(rid)
            orc.free(rid)
    return out


def run_schedule(S, cfg: synth.ModelConfig, reqs: Sequence[Tuple[int, int, int, int]], B: int, C: int,
                 num_blocks: int, block_size: int, weight_seed: int = 0, tok_seed: int = 1001,
                 max_tokens: int = 64, dump: bool = True, oracle_weights=None,
                 host_tensors=None) -> List[StepResult]:
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=max_tokens), seed=weight_seed, host_tensors=host_tensors)
    m.alloc_kv(num_blocks, block_size)
    steps, info = gpu_schedule(S, m, cfg, reqs, B, C, num_blocks, block_size, tok_seed, dump)
    m.close()
    w = oracle_weights if oracle_weights is not None else om.model_weights(cfg, weight_seed)
    return oracle_schedule(w, steps, info, num_blocks, block_size)


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

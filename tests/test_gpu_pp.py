"""Pipeline parallelism (§3.2, L1-19 §5.3): the layers split over
S stage handles on cuda:0 (stage s holds layers [L s / S, L (s+1) / S); the first embeds, the last
owns the final norm + LM head), each hybrid batch flowing stage to stage through
sarathi_stage_output -> sarathi_stage_input.  Every batch's logits and every layer's residual
(concatenated over the stages) against the unsharded fp64 oracle; slots bit-exact on every stage."""
import dataclasses

import numpy as np
import pytest

import synth
from tests import gpu_harness as gh
from oracle import model as om

pytestmark = pytest.mark.gpu
TOL = 2e-2
REGRESS = 8e-3


@pytest.fixture(scope="module")
def S():
    from paper_2308_16369_b200 import sarathi
    return sarathi


def run_pp(S, cfg, reqs, stages, B, C, num_blocks, block_size, weight_seed=0, max_tokens=64, tok_seed=1001):
    models = [S.Model(S.config_from(cfg, max_tokens), seed=weight_seed, pp_stage=s, pp_stages=stages)
              for s in range(stages)]
    for m in models:
        m.alloc_kv(num_blocks, block_size)
    sched = S.Scheduler(B, C, num_blocks, block_size)
    for r in reqs:
        sched.submit(*r)
    info = {r[0]: (r[1], r[2]) for r in reqs}
    V = cfg.vocab
    tok = lambda rid, pos, n=1: synth.tokens(tok_seed, rid, pos, n, V)
    out, pending_adm = [], []
    while not sched.done():
        plan, admitted = sched.next()
        for rid in admitted:
            for m in models:
                m.request_alloc(rid, sum(info[rid]))
        pending_adm += admitted
        if plan is None:
            sched.idle_step()
            continue
        pre, decs = plan
        prefill = (pre[0], pre[1], tok(pre[0], pre[1], pre[2])) if pre is not None else None
        decodes = [(rid, int(tok(rid, pos)[0]), pos) for rid, pos in decs]
        T = (pre[2] if pre else 0) + len(decs)
        logits = np.zeros((T, V), dtype=np.float32)
        hidden, slots = [], []
        for s, m in enumerate(models):
            if s > 0:
                ptr, t_prev = models[s - 1].stage_output()
                assert t_prev == T
                m.stage_input(ptr)
            last = s == stages - 1
            m.run_hybrid_batch(prefill, decodes, flags=S.RETURN_ALL_ROWS | S.DUMP_LAYERS,
                               logits_host=logits if last else None)
            hidden += [m.hidden(l, T) for l in range(len(range(cfg.n_layers * s // stages,
                                                                cfg.n_layers * (s + 1) // stages)))]
            slots.append(m.slot_mapping())
        fin = sched.complete()
        out.append(dict(plan=plan, prefill=prefill, decodes=decodes, logits=logits, hidden=hidden,
                        slots=slots[0], all_slots=slots, admitted=pending_adm, finished=fin))
        pending_adm = []
        for rid in fin:
            for m in models:
                m.request_free(rid)
    for m in models:
        m.close()
    return out, info


@pytest.mark.parametrize("stages", [2, 4])
def test_pp_stages_match_oracle(S, stages):
    cfg = dataclasses.replace(synth.TINY, name="tiny-L4", n_layers=4)
    reqs = [(1, 5, 12, 0), (2, 11, 12, 0), (3, 16, 12, 0), (0, 64, 4, 3)]
    steps, info = run_pp(S, cfg, reqs, stages, B=4, C=16, num_blocks=32, block_size=16)
    for st in steps:
        for sl in st["all_slots"]:
            assert np.array_equal(sl, st["all_slots"][0])
        assert len(st["hidden"]) == cfg.n_layers
    res = gh.oracle_schedule(om.model_weights(cfg, 0), steps, info, 32, 16)
    for r in res:
        assert np.array_equal(r.gpu_slots, r.ref_slots)
    errs = gh.worst_errors(res)
    print(f"PP {stages} stages worst errors", errs)
    assert errs["logits"] <= TOL and errs["hidden"] <= TOL, errs
    assert errs["logits"] <= REGRESS and errs["hidden"] <= REGRESS, errs


def test_pp_stage_errors(S):
    cfg = dataclasses.replace(synth.TINY, name="tiny-L4", n_layers=4)
    with pytest.raises(S.SarathiError):
        S.Model(S.config_from(cfg, 16), seed=0, pp_stage=2, pp_stages=2)     # stage out of range
    with pytest.raises(S.SarathiError):
        S.Model(S.config_from(cfg, 16), seed=0, pp_stage=0, pp_stages=5)     # more stages than layers
    m = S.Model(S.config_from(cfg, 16), seed=0, pp_stage=1, pp_stages=2)
    m.alloc_kv(8, 16)
    m.request_alloc(1, 16)
    with pytest.raises(S.SarathiError) as e:                                   # no stage input given
        m.run_hybrid_batch((1, 0, synth.tokens(1, 1, 0, 4, cfg.vocab)), [], flags=S.NO_LOGITS)
    assert e.value.code == S.ESTATE
    with pytest.raises(S.SarathiError):
        m.weight(0, 16, 0, 16)                                                 # embedding lives on stage 0
    m.close()

"""Tensor-parallel host logic on CPU with torch.distributed (gloo, world_size 2): the Megatron
sharding the library generates weights with (sarathi_shard_map) tiles every logical tensor exactly
once across ranks with the synth init scales, and the schedule / block tables every rank computes
independently are bit-identical (SPMD: no control messages needed)."""
import os
import random

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

WORLD = 2


def _ranges_tile(ranges, total):
    ranges = sorted(ranges)
    pos = 0
    for a, b in ranges:
        if a != pos:
            return False
        pos = b
    return pos == total


def _check_sharding(S, cfg, world, rank):
    """Returns this rank's shard description: {tensor: (tau, scale, base, rows, cols)}."""
    ccfg = S.config_from(cfg, 64)
    out = {}
    for layer in (0, cfg.n_layers - 1):
        for tensor in (0, 1, 2, 3):
            tau, sc, base, (rows, cols) = S.shard_map(ccfg, rank, world, layer, tensor)
            out[(layer, tensor)] = (tau, sc, base, rows, cols)
    for tensor in (16, 18):
        tau, sc, base, (rows, cols) = S.shard_map(ccfg, rank, world, 0, tensor)
        out[(0, tensor)] = (tau, sc, base, rows, cols)
    return out


def _worker(rank, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2308_16369_b200 import sarathi as S
        results = {}
        for name in ("tiny", "llama-13b", "llama2-70b"):
            cfg = synth.CONFIGS[name]
            w = WORLD if name != "llama2-70b" else WORLD
            mine = _check_sharding(S, cfg, w, rank)
            gathered = [None] * WORLD
            dist.all_gather_object(gathered, {k: (v[0].tolist(), v[1].tolist(), v[2].tolist(), v[3], v[4])
                                              for k, v in mine.items()})
            results[name] = gathered
        # SPMD schedule: every rank forms the same plans / block tables from the same inputs
        rnd = random.Random(1234)
        reqs = [(i, rnd.randint(1, 300), rnd.randint(0, 40), rnd.randint(0, 20)) for i in range(40)]
        s = S.Scheduler(8, 64, 400, 16)
        for r in reqs:
            s.submit(*r)
        plans, tables = [], {}
        while not s.done():
            plan, adm = s.next()
            for rid in adm:
                tables[rid] = s.block_table(rid).tolist()
            if plan is None:
                s.idle_step()
                continue
            plans.append(plan)
            s.complete()
        gathered = [None] * WORLD
        dist.all_gather_object(gathered, (plans, tables))
        results["sched"] = gathered
        if rank == 0:
            result_q.put(results)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gathered():
    from paper_2308_16369_b200 import build
    build.build(verbose=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid()).randint(0, 2000)
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("name", ["tiny", "llama-13b", "llama2-70b"])
def test_tp_shards_tile_logical_tensors(gathered, name):
    cfg = synth.CONFIGS[name]
    per_rank = gathered[name]
    for layer in (0, cfg.n_layers - 1):
        # group row ranges by generator tensor id across all ranks' QKV/O/gate-up/down shards
        by_tau = {}
        for rk in per_rank:
            for tensor in (0, 1, 2, 3):
                tau, sc, base, rows, cols = rk[(layer, tensor)]
                for t, s_, b in zip(tau, sc, base):
                    by_tau.setdefault(t, []).append((b, b + cols, s_))
        kinds = [synth.WQ, synth.WK, synth.WV, synth.WO, synth.WG, synth.WU, synth.WD]
        assert sorted(by_tau) == sorted(synth.layer_tau(layer, k) for k in kinds)
        for k in kinds:
            tau = synth.layer_tau(layer, k)
            shape = synth.tensor_shape(cfg, k)
            ranges = [(a, b) for a, b, _ in by_tau[tau]]
            assert _ranges_tile(ranges, int(np.prod(shape))), (name, layer, k)
            want = synth.weight_scale_f32(synth.tensor_sigma(cfg, k))
            assert all(np.float32(s_) == want for _, _, s_ in by_tau[tau])
    # vocab-parallel LM head tiles [V, H]; the embedding is replicated on every rank
    ranges = []
    for rk in per_rank:
        tau, sc, base, rows, cols = rk[(0, 18)]
        assert set(tau) == {synth.WLM_TAU}
        ranges += [(b, b + cols) for b in base]
    assert _ranges_tile(ranges, cfg.vocab * cfg.hidden)
    emb = [rk[(0, 16)][2] for rk in per_rank]
    assert all(e == emb[0] for e in emb)


def test_tp_schedule_identical_across_ranks(gathered):
    plans = gathered["sched"]
    assert plans[0] == plans[1]
    assert len(plans[0][0]) > 10

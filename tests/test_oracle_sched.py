"""Pins for oracle/sched.py and oracle/metrics.py: paper arithmetic (tests/golden), SPEC
examples, hand traces of the stated policy, brute force."""
import json
import os
import random

import pytest

from oracle import metrics as om
from oracle import sched as os_

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


def test_plan_chunks_examples():
    g = GOLD["chunking_example"]
    plan = os_.plan_chunks(g["P"], g["C"])
    assert len(plan) == g["num_chunks"] and all(n == 256 for _, n in plan)
    assert os_.plan_chunks(5, 2) == [(0, 2), (2, 2), (4, 1)]
    assert os_.plan_chunks(3, 8) == [(0, 3)]
    with pytest.raises(ValueError):
        os_.plan_chunks(0, 4)


def test_progressive_mask_example():
    # Fig. fig-attn-chunk-prefills: chunk size 4, second iteration covers queries 4..7
    rng = os_.chunk_key_ranges(4, 4)
    assert rng[0] == (0, 4) and rng[-1] == (0, 7)
    # over the three iterations every query sees exactly the keys <= itself
    seen = [r for s, n in os_.plan_chunks(12, 4) for r in os_.chunk_key_ranges(s, n)]
    assert seen == [(0, q) for q in range(12)]


def test_kv_reload_counts_by_enumeration():
    for P, C in [(1024, 256), (1000, 256), (4, 1), (7, 7), (50, 3)]:
        plan = os_.plan_chunks(P, C)
        # enumerate: every chunk j reads the KV of every token with index < its end
        brute = sum(1 for s, n in plan for t in range(P) if t < s + n)
        assert os_.kv_reload_tokens(plan) == brute
        # "first chunk loaded N times, second N-1 times, ..."
        N = len(plan)
        per_chunk_loads = [sum(1 for s2, n2 in plan if s2 + n2 > s) for s, n in plan]
        assert per_chunk_loads == list(range(N, 0, -1))
    assert os_.kv_reload_tokens(os_.plan_chunks(1024, 256)) == 256 * 4 * 5 // 2
    assert os_.kv_reload_tokens(os_.plan_chunks(4, 1)) == 10


def test_tile_adjust_and_balanced_pd_and_piggyback():
    g = GOLD["tile_adjust"]
    for B in (1, 4, 18, 27):
        p = os_.advise_chunk_size(g["C"], B)
        assert p == g["C"] - (B - 1) and (p + B - 1) % g["tile"] == 0
    with pytest.raises(ValueError):
        os_.advise_chunk_size(128, 200)
    for case in GOLD["balanced_pd"]["cases"]:
        v = os_.optimal_pd(case["C"], case["B"])
        assert v == case["C"] / 17
        assert abs(v - case["paper_pd"]) / case["paper_pd"] < 0.1  # paper's "~" sweep point
    with pytest.raises(ValueError):
        os_.optimal_pd(256, 1)
    g = GOLD["piggyback"]
    P = 4096
    assert round(P / os_.piggyback_capacity(P, g["C"], g["B"])) in (g["approx_divisor"], g["approx_divisor"] + 1)


def test_max_batch_size_formula():
    GiB, MiB = 1 << 30, 1 << 20
    assert os_.max_batch_size(20 * GiB, 0, 2048, MiB) == 10
    assert os_.max_batch_size(1, 2, 1024, 1) == 0
    # exact floor boundary
    assert os_.max_batch_size(100, 0, 10, 1) == 10 and os_.max_batch_size(99, 0, 10, 1) == 9


def test_block_allocator_lowest_first_vs_brute_force():
    rnd = random.Random(0)
    for trial in range(30):
        nb, bs = rnd.randint(1, 40), rnd.choice([1, 4, 16, 64])
        a = os_.BlockAllocator(nb, bs)
        free = [True] * nb
        owned = {}
        for step in range(60):
            if owned and rnd.random() < 0.4:
                rid = rnd.choice(sorted(owned))
                a.free(rid)
                for b in owned.pop(rid):
                    free[b] = True
                continue
            rid = 1000 * trial + step
            mt = rnd.randint(1, 6 * bs)
            need = -(-mt // bs)
            if need > sum(free):
                assert not a.can_alloc(mt)
                with pytest.raises(MemoryError):
                    a.alloc(rid, mt)
                continue
            got = a.alloc(rid, mt)
            exp = [i for i in range(nb) if free[i]][:need]
            assert got == exp
            for b in exp:
                free[b] = False
            owned[rid] = exp
            for pos in range(mt):
                assert a.slot(rid, pos) == exp[pos // bs] * bs + pos % bs


CONFIG1_EXPECTED = [
    # (prefill (req, start, n) or None, decodes [(req, pos)])  -- hand trace of O-16 policy
    ((1, 0, 5), []),
    ((2, 0, 11), [(1, 5)]),
    ((3, 0, 16), [(1, 6), (2, 11)]),
    ((0, 0, 16), [(1, 7), (2, 12), (3, 16)]),
    ((0, 16, 16), [(1, 8), (2, 13), (3, 17)]),
    ((0, 32, 16), [(1, 9), (2, 14), (3, 18)]),
    ((0, 48, 16), [(1, 10), (2, 15), (3, 19)]),
    (None, [(1, 11), (2, 16), (3, 20), (0, 64)]),
    (None, [(1, 12), (2, 17), (3, 21), (0, 65)]),
    (None, [(1, 13), (2, 18), (3, 22), (0, 66)]),
    (None, [(1, 14), (2, 19), (3, 23), (0, 67)]),
    (None, [(1, 15), (2, 20), (3, 24)]),
    (None, [(1, 16), (2, 21), (3, 25)]),
    (None, [(2, 22), (3, 26)]),
    (None, [(3, 27)]),
]


def config1_scheduler():
    alloc = os_.BlockAllocator(32, 16)
    s = os_.Scheduler(B=4, C=16, allocator=alloc)
    for rid, P, D, arr in [(1, 5, 12, 0), (2, 11, 12, 0), (3, 16, 12, 0), (0, 64, 4, 3)]:
        s.submit(rid, P, D, arr)
    return s, alloc


def test_config1_schedule_hand_trace():
    s, alloc = config1_scheduler()
    plans = []
    tables = {}
    while not s.done():
        p = s.next_batch()
        for rid in alloc.tables:
            tables.setdefault(rid, list(alloc.tables[rid]))
        plans.append(p)
        s.complete(p)
    assert [(p.prefill, p.decodes) for p in plans] == CONFIG1_EXPECTED
    assert tables == {1: [0, 1], 2: [2, 3], 3: [4, 5], 0: [6, 7, 8, 9, 10]}
    assert os_.slot_of(tables[0], 20, 16) == 7 * 16 + 4
    assert len(alloc.free_set) == 32


def test_spec_policy_examples():
    # one request prefilling (P=1024) + 3 decoding, C=256 tile-adjusted -> 253 + 3
    alloc = os_.BlockAllocator(1000, 16)
    s = os_.Scheduler(B=4, C=256, allocator=alloc, tile_adjust=True)
    for rid in (1, 2, 3):
        s.submit(rid, 1, 100, 0)
    s.complete(s.next_batch()); s.complete(s.next_batch()); s.complete(s.next_batch())
    s.submit(9, 1024, 10, 0)
    p = s.next_batch()
    assert p.prefill == (9, 0, 253) and len(p.decodes) == 3
    # no prefill pending, 5 decoders, B=8 -> decode-only batch of 5
    alloc = os_.BlockAllocator(1000, 16)
    s = os_.Scheduler(B=8, C=256, allocator=alloc)
    for rid in range(5):
        s.submit(rid, 1, 100, 0)
    for _ in range(5):
        s.complete(s.next_batch())
    p = s.next_batch()
    assert p.prefill is None and len(p.decodes) == 5


def test_orca_best_is_sarathi_with_full_prompt():
    alloc = os_.BlockAllocator(100, 16)
    s = os_.Scheduler(B=4, C=256, allocator=alloc, policy=os_.ORCA_BEST)
    s.submit(0, 700, 2, 0)
    assert s.next_batch().prefill == (0, 0, 700)


def test_request_level_never_mixes():
    alloc = os_.BlockAllocator(100, 16)
    s = os_.Scheduler(B=2, C=256, allocator=alloc, policy=os_.REQUEST_LEVEL)
    for rid, arr in [(0, 0), (1, 0), (2, 0)]:
        s.submit(rid, 40, 3, arr)
    plans = os_.run_schedule(s)
    for p in plans:
        assert p.prefill is None or not p.decodes
    assert plans[0].prefill == (0, 0, 40) and plans[1].prefill == (1, 0, 40)
    # request 2 only after the first cohort drained
    first2 = next(i for i, p in enumerate(plans) if p.prefill and p.prefill[0] == 2)
    assert all(not (p.decodes and any(r in (0, 1) for r, _ in p.decodes)) for p in plans[first2:])


@pytest.mark.parametrize("seed", range(5))
def test_sarathi_schedule_properties(seed):
    rnd = random.Random(seed)
    B, C, bs = rnd.randint(2, 6), rnd.choice([4, 16, 32]), rnd.choice([4, 16])
    alloc = os_.BlockAllocator(rnd.randint(20, 80), bs)
    s = os_.Scheduler(B, C, alloc)
    reqs = {}
    for rid in range(rnd.randint(3, 12)):
        P, D = rnd.randint(1, 60), rnd.randint(0, 20)
        if -(-(P + D) // bs) > alloc.num_blocks:
            continue
        reqs[rid] = (P, D)
        s.submit(rid, P, D, rnd.randint(0, 10))
    plans = os_.run_schedule(s)
    seen_pos = {r: 0 for r in reqs}
    prefill_order = []
    for p in plans:
        assert p.num_tokens >= 1
        ids = [r for r, _ in p.decodes] + ([p.prefill[0]] if p.prefill else [])
        assert len(ids) == len(set(ids))
        if p.prefill:
            assert len(p.decodes) <= B - 1
            rid, st, n = p.prefill
            assert st == seen_pos[rid] and 1 <= n <= C
            seen_pos[rid] += n
            if not prefill_order or prefill_order[-1] != rid:
                prefill_order.append(rid)
        else:
            assert len(p.decodes) <= B
        for rid, pos in p.decodes:
            assert pos == seen_pos[rid] and pos >= reqs[rid][0]
            seen_pos[rid] += 1
    assert all(seen_pos[r] == P + D for r, (P, D) in reqs.items())
    assert len(prefill_order) == len(set(prefill_order))  # each prompt served contiguously, FCFS
    assert len(alloc.free_set) == alloc.num_blocks


def test_paper_metric_arithmetic():
    t = GOLD["table_compute_split"]
    pm, do, pf = t["decode_maximal"], t["decode_only"], t["prefill_only"]
    assert abs(om.marginal_decode_time(pm["total_ms"], pf["total_ms"], pm["decodes"]) - pm["per_token_decode_ms"]) < 1e-9
    assert abs(om.baseline_decode_time(do["total_ms"], do["decodes"]) - do["per_token_decode_ms"]) < 1e-9
    assert abs(pf["total_ms"] / pf["prefill_tokens"] - pf["per_token_prefill_ms"]) < 5e-4
    assert abs(pf["linear_ms"] + pf["attn_ms"] - pf["total_ms"]) < 1e-9
    sp = om.decode_speedup(do["total_ms"], do["decodes"], pm["total_ms"], pf["total_ms"], pm["decodes"])
    assert 10.3 < sp < 10.5   # "an order of magnitude"
    assert om.hybrid_tokens_per_s(256, 64, 0.01) == 32000.0

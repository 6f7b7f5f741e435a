"""CPU tests of the C-ABI library: it loads, exports every symbol include/sarathi.h declares,
rejects bad arguments, and its host scheduler / block allocator match the oracle's independent
Python implementation bit-exactly (no GPU compute is called here)."""
import os
import random
import re

import pytest

from oracle import sched as osch
from tests.test_oracle_sched import CONFIG1_EXPECTED

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "sarathi.h")


@pytest.fixture(scope="module")
def S():
    from paper_2308_16369_b200 import build
    build.build(verbose=False)
    from paper_2308_16369_b200 import sarathi
    return sarathi


def test_library_exports_every_header_symbol(S):
    text = open(HEADER).read()
    declared = sorted(set(re.findall(r"\b(sarathi_[a-z_0-9]+)\s*\(", text)))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(S.lib, name), name
    assert sorted(S.EXPORTS) == declared


def test_error_reporting_without_gpu(S):
    with pytest.raises(S.SarathiError) as e:
        S.Scheduler(0, 16, 10, 16)
    assert e.value.code == S.EINVAL and "sched_create" in str(e.value)
    with pytest.raises(S.SarathiError):
        S.Scheduler(4, 3, 10, 16, tile_adjust=True)  # C-(B-1) = 0
    s = S.Scheduler(4, 16, 10, 16)
    s.submit(1, 5, 1)
    with pytest.raises(S.SarathiError) as e:
        s.submit(1, 5, 1)
    assert e.value.code == S.EINVAL


def test_never_admissible_request_is_rejected_at_submit(S):
    """A request whose P+D reservation exceeds the whole pool could never be admitted; under strict
    FCFS it would block every later request forever.  Both schedulers refuse it at submit (C++:
    ENOKV, Python twin: ValueError) and the later requests still drain."""
    s = S.Scheduler(2, 16, 4, 16)                  # pool: 4 blocks x 16 tokens = 64 tokens
    with pytest.raises(S.SarathiError) as e:
        s.submit(1, 60, 5)                          # 65 tokens -> 5 blocks > 4
    assert e.value.code == S.ENOKV
    with pytest.raises(S.SarathiError) as e:
        s.submit(2, 2 ** 31 - 1, 2 ** 31 - 1)       # P+D overflows int32: still rejected, not wrapped
    assert e.value.code == S.ENOKV
    s.submit(3, 40, 24)                             # exactly 64 tokens: admissible
    plans, _ = _drain_cpp_sched(s)
    assert plans and s.done()
    py = osch.Scheduler(2, 16, osch.BlockAllocator(4, 16))
    with pytest.raises(ValueError):
        py.submit(1, 60, 5)
    py.submit(3, 40, 24)
    assert osch.run_schedule(py)


def test_sched_cap_checked_before_state_changes(S):
    """sched_next / sched_complete with cap < B fail with EINVAL and leave the scheduler as it was
    (the admitted ids and finished ids would otherwise be lost)."""
    s = S.Scheduler(4, 16, 32, 16)
    for rid in range(3):
        s.submit(rid, 8, 1)
    cap, s.cap = s.cap, 3                           # 3 < B = 4
    with pytest.raises(S.SarathiError) as e:
        s.next()
    assert e.value.code == S.EINVAL
    s.cap = cap
    plan, admitted = s.next()                       # nothing was admitted by the failed call
    assert admitted == [0, 1, 2] and plan[0] == (0, 0, 8)
    s.cap = 2
    with pytest.raises(S.SarathiError):
        s.complete()
    s.cap = cap
    assert s.complete() == []                       # the plan is still pending, completes once
    plan, admitted = s.next()
    assert admitted == [] and plan[0] == (1, 0, 8) and plan[1] == [(0, 8)]


def test_host_tensors_count_checked_before_the_library(S):
    import synth
    with pytest.raises(ValueError):
        S.Model(S.config_from(synth.TINY, 16), seed=0, host_tensors=[None] * 5)


def _drain_cpp_sched(s):
    plans = []
    while not s.done():
        plan, _ = s.next()
        if plan is None:
            s.idle_step()
            continue
        plans.append(plan)
        s.complete()
    return plans, None


def _drain_cpp(S, B, C, nb, bs, reqs, policy=0, tile_adjust=False):
    s = S.Scheduler(B, C, nb, bs, policy=policy, tile_adjust=tile_adjust)
    for rid, P, D, arr in reqs:
        s.submit(rid, P, D, arr)
    plans, tables = [], {}
    guard = 0
    while not s.done():
        guard += 1
        assert guard < 100000
        plan, admitted = s.next()
        for rid in admitted:
            tables[rid] = list(s.block_table(rid))
        if plan is None:
            s.idle_step()
            continue
        plans.append(plan)
        s.complete()
    return plans, tables


def _drain_py(B, C, nb, bs, reqs, policy=osch.SARATHI, tile_adjust=False):
    alloc = osch.BlockAllocator(nb, bs)
    s = osch.Scheduler(B, C, alloc, policy=policy, tile_adjust=tile_adjust)
    for rid, P, D, arr in reqs:
        s.submit(rid, P, D, arr)
    plans, tables = [], {}
    while not s.done():
        p = s.next_batch()
        for rid, t in alloc.tables.items():
            tables.setdefault(rid, list(t))
        if p is None:
            s.idle_step()
            continue
        plans.append((p.prefill, p.decodes))
        s.complete(p)
    return plans, tables


def test_cpp_scheduler_config1_hand_trace(S):
    reqs = [(1, 5, 12, 0), (2, 11, 12, 0), (3, 16, 12, 0), (0, 64, 4, 3)]
    plans, tables = _drain_cpp(S, 4, 16, 32, 16, reqs)
    assert plans == CONFIG1_EXPECTED
    assert tables == {1: [0, 1], 2: [2, 3], 3: [4, 5], 0: [6, 7, 8, 9, 10]}


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("policy", [0, 1, 2])
def test_cpp_scheduler_matches_python_twin(S, seed, policy):
    rnd = random.Random(seed * 7 + policy)
    B, C, bs = rnd.randint(1, 8), rnd.choice([4, 16, 64, 256]), rnd.choice([16, 64])
    nb = rnd.randint(8, 200)
    tile = rnd.choice([0, 0, 1, 2]) if policy == 0 else 0
    if tile == 1 and C <= B - 1:
        tile = 0
    reqs = []
    for rid in range(rnd.randint(1, 25)):
        P, D = rnd.randint(1, 300), rnd.randint(0, 40)
        if -(-(P + D) // bs) > nb:
            continue
        reqs.append((rid * 3 + 1, P, D, rnd.randint(0, 30)))
    py_policy = [osch.SARATHI, osch.ORCA_BEST, osch.REQUEST_LEVEL][policy]
    a = _drain_cpp(S, B, C, nb, bs, reqs, policy, tile)
    b = _drain_py(B, C, nb, bs, reqs, py_policy, tile)
    assert a[0] == b[0]
    assert a[1] == b[1]


def test_b200_chunk_advisor_hand_cases_and_cpp_twin(S):
    """B200 tile-quantization chunk rule (PAPER.md L457-463 restated on the tcgen05 GEMM's token
    quanta): hand-computed cases, then the C++ advisor / token tiling == the Python twin."""
    cap = osch.gemm_token_capacity
    # token capacity: 16-multiples up to 256 (one UMMA), 32-multiples to 512 (two), then 2 tiles
    assert [cap(t) for t in (1, 16, 17, 255, 256, 257, 288, 289, 320, 512, 513, 1024)] == \
        [16, 16, 32, 256, 256, 288, 288, 320, 320, 512, 576, 1024]
    ch = osch.b200_chunk
    assert ch(256, 0, 10**6) == 256          # exactly on the quantum
    assert ch(256, 1, 10**6) == 287          # 257 tokens: no step at 256 any more, fill the 288-token tile
    assert ch(256, 32, 10**6) == 256         # T = 288 = capacity
    assert ch(256, 33, 10**6) == 287         # T = 289: fill the 320-token tile
    assert ch(256, 64, 10**6) == 256         # T = 320 = capacity
    assert ch(128, 5, 10**6) == 139          # T = 133 -> 144-token tile: fill
    assert ch(128, 5, 50) == 50              # the last chunk of a prompt
    assert ch(500, 20, 10**6) == 492         # T = 520 overshoots 512 by 8 <= 62: trim
    for C in (16, 64, 128, 192, 256, 320, 384, 512):
        for d in range(0, 140, 3):
            for rem in (1, 7, C // 2 + 1, 10**6):
                assert S.chunk_advice(C, d, rem) == osch.b200_chunk(C, d, rem), (C, d, rem)
    for T in range(1, 1600):
        assert S.token_capacity(T)[0] == cap(T), T


def test_library_sass_is_blackwell_native(S):
    """The built library runs on sm_100a tensor-core / TMA / TMEM instructions (tcgen05.mma ->
    UTCHMMA incl. the CTA-pair form, cp.async.bulk.tensor -> UTMALDG, tcgen05.ld -> LDTM) and
    the NVLS all-reduce consumer compiles to multimem.ld_reduce (LDGMC)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", S.LIB_PATH], capture_output=True, text=True).stdout
    for op in ("UTCHMMA.2CTA", "UTMALDG.2D.2CTA", "LDTM", "LDGMC"):
        assert op in sass, op
    assert "sm_100a" in subprocess.run([exe, "-lelf", S.LIB_PATH], capture_output=True, text=True).stdout


def test_pipeline_timeline_hand_cases():
    """Max-plus pipeline recurrence (paper_2308_16369_b200/pipeline.py) on hand-worked cases: uniform
    micro-batches leave no bubble; a long first micro-batch (a full prompt, PB1) stalls its slot's
    next iteration: stage 0 idles 2 units before micro-batch 2 (t = [3, 1, 1, 1], 2 stages)."""
    from paper_2308_16369_b200.pipeline import pipeline_timeline, request_bubbles
    _, fin, bub = pipeline_timeline([1, 1, 1, 1], 2)
    assert bub == [0, 0, 0, 0] and fin[1][3] == 5
    st, fin, bub = pipeline_timeline([3, 1, 1, 1], 2)
    assert bub == [0, 0, 2, 0]
    assert [st[0][m] for m in range(4)] == [0, 3, 6, 7] and [fin[1][m] for m in range(4)] == [6, 7, 8, 9]
    assert request_bubbles([[1, 2], [3], [1], [3]], bub) == {1: 2.0, 2: 0.0, 3: 0.0}
    _, fin, bub = pipeline_timeline([2, 5], 1)          # one stage: no pipeline, no bubbles
    assert bub == [0, 0] and fin[0][1] == 7

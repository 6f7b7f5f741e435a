"""Layer-chain work list (host_sched.cpp schedule_chain via the C ABI, no GPU): every unit of
every job is executed exactly once (a whole-tile job's tile may be split; its contributors then
reduce through a scratch slab), a pair runs its segments in job order (the dependency graph of the
one-launch chain is then acyclic), and the predicted makespan is within a small factor of the
work bound on the LLaMA-13B layer chain and a TP-8 rank's small-M chain."""
import numpy as np
import pytest

from paper_2308_16369_b200 import sarathi as S


def _check_cover(jobs, off, segs):
    seen = [np.zeros((pm, kb), np.int32) for pm, kb, *_ in jobs]
    for c in range(len(off) - 1):
        last_job = -1
        for j, pt, k0, k1 in segs[off[c]:off[c + 1]]:
            assert j >= last_job, "pair runs its segments in job order"
            last_job = j
            pm, KB = jobs[j][0], jobs[j][1]
            assert 0 <= pt < pm and 0 <= k0 < k1 <= KB
            seen[j][pt, k0:k1] += 1
    for s in seen:
        assert (s == 1).all(), "every (tile, k-block) unit exactly once"


def test_hand_case_water_filling():
    # 2 pairs; job 0: 2 whole tiles of 10 k-blocks (one per pair, ends at 10);
    # job 1: one split tile of 20 k-blocks, no dependency -> 10 each, makespan 20
    jobs = [(2, 10, 0, -1, 0.0), (1, 20, 1, -1, 0.0)]
    off, segs, ms = S.chain_schedule(jobs, 2, 0.0, 0.0)
    _check_cover(jobs, off, segs)
    assert ms == pytest.approx(20.0)
    assert sorted(tuple(s) for s in segs[segs[:, 0] == 1]) == [(1, 0, 0, 10), (1, 0, 10, 20)]


def test_hand_case_dependency_wait():
    # job 1's k-block kb needs job 0's 128-row tile kb (shift 0); job 0 publishes at 10 + 5.
    # Water-filling folds its 2-unit ranges (below min_seg = 4) into one pair (15 + 4 = 19); the
    # tile-aligned split in 2 parts keeps one segment per pair: 15 + 2 = 17, and is kept
    jobs = [(2, 10, 0, -1, 5.0), (1, 4, 1, 0, 0.0)]
    off, segs, ms = S.chain_schedule(jobs, 2, 0.0, 0.0)
    _check_cover(jobs, off, segs)
    assert ms == pytest.approx(17.0)
    assert sorted(tuple(s) for s in segs[segs[:, 0] == 1]) == [(1, 0, 0, 2), (1, 0, 2, 4)]


@pytest.mark.parametrize("swiglu", [True, False])
def test_llama13b_layer_chain(swiglu):
    H, H2, qkv = 5120, 13824, 15360
    gu = 2 * H2 if swiglu else H2
    jobs = [(H // 256, H // 64, 1, -1, 0.0), (gu // 256, H // 64, 0, 1, 18.0),
            (H // 256, H2 // 64, 1, 0 if swiglu else 1, 0.0), (qkv // 256, H // 64, 0, 1, 30.0)]
    off, segs, ms = S.chain_schedule(jobs, 74, 8.0, 4.0)
    _check_cover(jobs, off, segs)
    work = sum(pm * kb for pm, kb, *_ in jobs) / 74
    assert work <= ms <= 1.5 * work + 60, (ms, work)
    # at most ~16 contributors per tile and band (each costs a partial reduction)
    for j in range(4):
        _, counts = np.unique(segs[segs[:, 0] == j][:, 1], return_counts=True)
        assert counts.max() <= 32


def test_small_m_rank_chain_splits_tiles():
    # LLaMA-2-70B TP-8 rank: QKV has 5 pair tiles of 128 k-blocks; whole tiles would leave 69 of
    # 74 pairs idle, so the schedule must split them
    jobs = [(32, 16, 1, -1, 0.0), (28, 128, 0, 1, 22.0), (32, 56, 1, 0, 0.0), (5, 128, 0, 1, 27.0)]
    off, segs, ms = S.chain_schedule(jobs, 74, 16.0, 6.0)
    _check_cover(jobs, off, segs)
    qkv = segs[segs[:, 0] == 3]
    assert len(qkv) > 5 * 4, "QKV tiles split over many pairs"
    work = sum(pm * kb for pm, kb, *_ in jobs) / 74
    assert ms <= 3 * work + 150, (ms, work)


def test_random_chains_cover():
    rng = np.random.default_rng(5)
    for _ in range(40):
        nj = int(rng.integers(1, 5))
        jobs = []
        for j in range(nj):
            jobs.append((int(rng.integers(1, 30)), int(rng.integers(1, 90)), int(rng.integers(0, 2)),
                         -1 if j == 0 else int(rng.integers(-1, 3)), float(rng.uniform(0, 20))))
        pairs = int(rng.integers(1, 80))
        off, segs, ms = S.chain_schedule(jobs, pairs, 3.0, 2.0)
        _check_cover(jobs, off, segs)
        assert ms >= sum(pm * kb for pm, kb, *_ in jobs) / pairs - 1e-9

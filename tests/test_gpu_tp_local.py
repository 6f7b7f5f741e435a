"""Tensor parallelism on ONE GPU (§2.3 Megatron TP): a local group of
`world` model handles on cuda:0, one host thread per rank making identical calls, runs every
world > 1 path of the library — column-parallel QKV / gate||up and row-parallel O / down shards,
bf16 partials + all-reduce (2 per layer) fused into the next RMSNorm, the last layer's pending
partial, the vocab-parallel LM head + all-gather + permute — against the UNSHARDED fp64 oracle.

Checks per schedule: every rank returns bit-identical logits and per-layer residuals (SPMD: the
all-reduce result is identical everywhere), slot mappings are bit-exact, and logits / residuals
are within the 2e-2 contract (8e-3 regression bound) of the oracle."""
import dataclasses
import os
import threading

import numpy as np
import pytest

import synth
from oracle import model as om
from tests import gpu_harness as gh

pytestmark = pytest.mark.gpu
TOL = 2e-2
REGRESS = 8e-3


@pytest.fixture(scope="module")
def S():
    from paper_2308_16369_b200 import sarathi
    return sarathi


def run_tp(S, cfg, reqs, world, B, C, num_blocks, block_size, weight_seed=0, max_tokens=64, host_tensors=None,
           fused=True):
    """fused: the NEXT-1 path (one-shot all-reduce fused into the consuming RMSNorm over peer
    memory, ready flags + double-buffered partials); else the summing-kernel stand-in for NCCL."""
    g = S.LocalGroup(world)
    old = os.environ.get("SARATHI_TP_FUSED")
    os.environ["SARATHI_TP_FUSED"] = "1" if fused else "0"
    try:
        models = [S.Model(S.config_from(cfg, max_tokens), seed=weight_seed, rank=r, world=world, local_group=g,
                          host_tensors=host_tensors) for r in range(world)]
    finally:
        if old is None:
            os.environ.pop("SARATHI_TP_FUSED")
        else:
            os.environ["SARATHI_TP_FUSED"] = old
    for m in models:
        m.alloc_kv(num_blocks, block_size)
    res = [None] * world

    def work(r):
        try:
            res[r] = gh.gpu_schedule(S, models[r], cfg, reqs, B, C, num_blocks, block_size)
        except BaseException as e:  # noqa: BLE001 - re-raised below on the main thread
            res[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for m in models:
        m.close()
    g.close()
    for r in res:
        if isinstance(r, BaseException):
            raise r
    return res


def _check_tp(res, cfg, weight_seed, num_blocks, block_size):
    steps0, info = res[0]
    for r, (steps, _) in enumerate(res[1:], 1):
        assert len(steps) == len(steps0)
        for a, b in zip(steps0, steps):
            assert a["plan"] == b["plan"]
            assert np.array_equal(a["slots"], b["slots"])
            assert np.array_equal(a["logits"], b["logits"]), f"rank {r} logits differ from rank 0"
            for ha, hb in zip(a["hidden"], b["hidden"]):
                assert np.array_equal(ha, hb), f"rank {r} residual differs from rank 0"
    w = om.model_weights(cfg, weight_seed)
    steps = gh.oracle_schedule(w, steps0, info, num_blocks, block_size)
    for s in steps:
        assert np.array_equal(s.gpu_slots, s.ref_slots)
    errs = gh.worst_errors(steps)
    print(f"{cfg.name} world={len(res)} worst errors", errs)
    if errs["logits"] > REGRESS or errs["hidden"] > REGRESS:
        for i, s in enumerate(steps):
            print(" step", i, s.plan, gh.worst_errors([s]),
                  [float(np.max(np.abs(g - r)) / np.max(np.abs(r))) for g, r in zip(s.gpu_hidden, s.ref_hidden)])
    assert errs["logits"] <= TOL and errs["hidden"] <= TOL, errs
    assert errs["logits"] <= REGRESS and errs["hidden"] <= REGRESS, errs
    return errs


CONFIG1 = [(1, 5, 12, 0), (2, 11, 12, 0), (3, 16, 12, 0), (0, 64, 4, 3)]


@pytest.mark.parametrize("fused", [True, False], ids=["fused-ar", "sum-kernel"])
@pytest.mark.parametrize("world", [2, 4])
def test_tp_tiny_config1(S, world, fused):
    res = run_tp(S, synth.TINY, CONFIG1, world, B=4, C=16, num_blocks=32, block_size=16, fused=fused)
    _check_tp(res, synth.TINY, 0, 32, 16)


@pytest.mark.parametrize("case", ["gqa-bs64", "gqa-bs16", "gelu", "gelu-host"])
def test_tp_gqa_gelu_and_host_weights(S, case):
    """GQA (KV heads sharded, 1 per rank at world 2, group 2) and the GELU 2-matrix FFN (W1
    column-, W2 row-parallel), the latter also with weights uploaded from host memory (host_tensors
    sharded by the library)."""
    if case.startswith("gqa"):
        cfg = dataclasses.replace(synth.TINY, name="tiny-gqa", n_kv_heads=2, max_seq_len=256)
        bs = 64 if case == "gqa-bs64" else 16
        reqs = [(5, 70, 6, 0), (6, 3, 20, 0), (7, 130, 3, 2)]
        res = run_tp(S, cfg, reqs, 2, B=3, C=32, num_blocks=16 * (64 // bs), block_size=bs, weight_seed=3)
        _check_tp(res, cfg, 3, 16 * (64 // bs), bs)
    else:
        cfg = dataclasses.replace(synth.TINY, name="tiny-gelu", ffn_kind=synth.FFN_GELU, ffn_hidden=1024)
        ht = gh.synth_host_tensors(cfg, 5) if case == "gelu-host" else None
        res = run_tp(S, cfg, [(1, 20, 5, 0), (2, 9, 7, 0)], 2, B=2, C=8, num_blocks=16, block_size=16, weight_seed=5,
                     host_tensors=ht)
        _check_tp(res, cfg, 5, 16, 16)


@pytest.mark.parametrize("fused", [True, False], ids=["fused-ar", "sum-kernel"])
@pytest.mark.parametrize("world", [2, 4])
def test_tp_llama13b_width_two_layers(S, world, fused):
    """LLaMA-13B width (H 5120, 40 heads, H2 13824, V 32000), 2 layers, TP 2 / 4: rank shards of
    the real shapes (TP4: 10 heads, 3456 FFN rows, 8000 vocab rows per rank) against the unsharded
    oracle; a chunked prompt with decodes riding along."""
    cfg = dataclasses.replace(synth.LLAMA_13B, name="llama13b-L2", n_layers=2, max_seq_len=512)
    reqs = [(1, 40, 3, 0), (2, 150, 2, 0)]
    res = run_tp(S, cfg, reqs, world, B=2, C=64, num_blocks=16, block_size=64, max_tokens=80, fused=fused)
    _check_tp(res, cfg, 0, 16, 64)


@pytest.mark.parametrize("variant", ["gqa", "gelu"])
def test_tp_host_tensor_shards_bit_identical(S, variant):
    """Each rank's packed shard loaded from host_tensors equals, bit for bit, the shard the seed path
    generates on device for the same rank (sarathi_shard_map rows of the logical tensors)."""
    if variant == "gqa":
        cfg = dataclasses.replace(synth.TINY, name="tiny-gqa", n_kv_heads=2)
    else:
        cfg = dataclasses.replace(synth.TINY, name="tiny-gelu", ffn_kind=synth.FFN_GELU, ffn_hidden=1024)
    world = 2
    ht = gh.synth_host_tensors(cfg, 5)
    ga, gb = S.LocalGroup(world), S.LocalGroup(world)
    H = cfg.hidden
    for r in range(world):
        a = S.Model(S.config_from(cfg, 16), seed=5, rank=r, world=world, local_group=ga)
        b = S.Model(S.config_from(cfg, 16), seed=0, rank=r, world=world, local_group=gb, host_tensors=ht)
        for t in (0, 1, 2, 3, 16, 18):
            _, _, _, (rows, cols) = S.shard_map(S.config_from(cfg, 16), r, world, 0, t)
            for l in (range(cfg.n_layers) if t < 16 else [0]):
                wa, wb = a.weight(l, t, 0, rows * cols), b.weight(l, t, 0, rows * cols)
                assert np.array_equal(wa, wb), (r, l, t, int(np.sum(wa != wb)))
        for l in range(cfg.n_layers):
            for t in (4, 5):
                assert np.array_equal(a.weight(l, t, 0, H), b.weight(l, t, 0, H)), (r, l, t)
        a.close()
        b.close()
    ga.close()
    gb.close()

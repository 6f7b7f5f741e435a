"""Pins for the seeded input generator (synth): known hash vectors, library bf16 rounding,
distribution statistics, the paper's workload recipe."""
import math

import numpy as np
import pytest
import torch

import synth


def test_splitmix64_known_vectors():
    # Reference outputs of the splitmix64 finaliser (Vigna's SplitMix64, state 0 / 1 / 2 steps):
    # the first three outputs of a SplitMix64 generator seeded with 0 are these constants.
    expected = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    outs = [synth.splitmix64_scalar((i * synth.GOLDEN) & synth.MASK64) for i in range(3)]
    assert outs == expected


def test_splitmix64_vectorised_equals_scalar():
    xs = np.array([0, 1, 2, 12345, (1 << 63) + 7, synth.MASK64], dtype=np.uint64)
    v = synth.splitmix64(xs)
    for x, y in zip(xs.tolist(), v.tolist()):
        assert synth.splitmix64_scalar(int(x)) == int(y)


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 3,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.0039062 + 1e-7, -2.5e-30, 6.5e4], np.float32)])
    ours = synth.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    back = synth.bf16_bits_to_f32(ours)
    assert np.array_equal(back, torch.from_numpy(x).to(torch.bfloat16).float().numpy())


def test_weight_distribution_uniform_with_sigma():
    cfg = synth.TINY
    w = synth.as_f64(synth.layer_tensor_bits(cfg, 0, 0, synth.WQ))
    sig = synth.tensor_sigma(cfg, synth.WQ)
    assert abs(w.mean()) < 0.01 * sig
    assert abs(w.std() / sig - 1.0) < 0.01
    assert np.max(np.abs(w)) <= math.sqrt(3) * sig * (1 + 2 ** -8)


def test_gains_near_one_and_tensors_differ():
    cfg = synth.TINY
    g = synth.as_f64(synth.layer_tensor_bits(cfg, 0, 1, synth.G1))
    assert np.all(np.abs(g - 1.0) <= 0.1 + 2 ** -7)
    a = synth.layer_tensor_bits(cfg, 0, 0, synth.WK)
    b = synth.layer_tensor_bits(cfg, 0, 0, synth.WV)
    c = synth.layer_tensor_bits(cfg, 1, 0, synth.WK)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_rows_helpers_match_full_tensor():
    cfg = synth.TINY
    full = synth.layer_tensor_bits(cfg, 3, 1, synth.WD)
    rows = synth.layer_tensor_rows_bits(cfg, 3, 1, synth.WD, [0, 5, 255])
    assert np.array_equal(full[[0, 5, 255]], rows)
    e = synth.embedding_bits(cfg, 3)
    assert np.array_equal(e[[7, 9]], synth.embedding_rows_bits(cfg, 3, [7, 9]))
    lm = synth.lm_head_bits(cfg, 3)
    assert np.array_equal(lm[[1, 511]], synth.lm_head_rows_bits(cfg, 3, [1, 511]))


def test_tokens_in_range_and_uniform():
    t = synth.tokens(11, 3, 0, 200000, 512)
    assert t.min() >= 0 and t.max() < 512
    counts = np.bincount(t, minlength=512)
    chi2 = ((counts - counts.mean()) ** 2 / counts.mean()).sum()
    assert chi2 < 512 + 6 * math.sqrt(2 * 512)
    assert np.array_equal(synth.tokens(11, 3, 100, 10, 512), t[100:110])


@pytest.mark.parametrize("theta", [0.0, 0.4, 1.0])
def test_zipf_chi_square(theta):
    lo, hi, n = 1, 8, 200000
    lens = synth.zipf_lengths(5, n, lo, hi, theta)
    ranks = np.arange(1, hi - lo + 2, dtype=np.float64)
    p = ranks ** (-theta)
    p /= p.sum()
    counts = np.bincount(lens - lo, minlength=hi - lo + 1)
    chi2 = ((counts - n * p) ** 2 / (n * p)).sum()
    assert chi2 < 30.0  # 7 dof; p ~ 1e-4


def test_zipf_paper_range_and_orientation():
    lens = synth.zipf_lengths(1, 20000)  # 1K..4K, theta 0.4
    assert lens.min() >= 1024 and lens.max() <= 4096
    # rank 1 = shortest => the lower half of the range is more likely
    assert (lens < 2560).mean() > 0.5


def test_split_pd_examples():
    assert synth.split_pd(1100, 10) == (1000, 100)
    assert synth.split_pd(2, 50) == (1, 1)
    p, d = synth.split_pd(3000, 1)
    assert (p, d) == (1500, 1500)
    w = synth.zipf_workload(4, 50, 10.0)
    assert all(r.prompt_len + r.decode_len >= 1024 for r in w)

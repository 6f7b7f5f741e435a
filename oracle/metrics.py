"""The paper's throughput metrics — TEST INFRASTRUCTURE ONLY (also used by bench.py's
cpu_baseline leg).

P:L32 (§5.1.1): "we find the difference in runtime between the decode-maximal batch and a
prefill-only batch of prefill size p, and attribute the difference in time as the marginal
decode time for a batch of d requests"; the baseline "dividing the time to process one decode
iteration by the batch size".  Table tbl-compute-split instantiates both.
"""
from __future__ import annotations


def marginal_decode_time(t_hybrid: float, t_prefill_only: float, d: int) -> float:
    if d <= 0:
        raise ValueError("d >= 1")
    return (t_hybrid - t_prefill_only) / d


def baseline_decode_time(t_decode_only: float, d: int) -> float:
    if d <= 0:
        raise ValueError("d >= 1")
    return t_decode_only / d


def decode_speedup(t_decode_only: float, d_decode_only: int, t_hybrid: float, t_prefill_only: float,
                   d_hybrid: int) -> float:
    return baseline_decode_time(t_decode_only, d_decode_only) / marginal_decode_time(t_hybrid, t_prefill_only, d_hybrid)


def hybrid_tokens_per_s(p: int, d: int, t_iter_s: float) -> float:
    return (p + d) / t_iter_s


def relative_error(gpu, ref) -> float:
    """||gpu - ref||_inf / ||ref||_inf  (reading O-20)."""
    import numpy as np
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(gpu - ref)) / (den if den > 0 else 1.0))

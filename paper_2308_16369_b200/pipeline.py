"""Pipeline-parallel timeline of micro-batches (host logic; §3.2 "pipeline
bubbles", L1-19 §5.3).

S stages, each holding L/S consecutive layers; micro-batches enter stage 0 in order m = 0, 1, ...;
micro-batch m belongs to in-flight slot m mod S (the S micro-batches in flight are disjoint request
groups, Orca-style PP) and its requests' next iteration (micro-batch m + S) can only start once m
has left the last stage (its tokens are needed).  With t[m] the per-stage time of micro-batch m:

    start[s][m]  = max(finish[s-1][m], finish[s][m-1], (s == 0) * finish[S-1][m-S])
    finish[s][m] = start[s][m] + t[m]

The bubble before micro-batch m on stage s is start[s][m] - finish[s][m-1] (the stage idles); the
paper's per-request bubble time is the sum of those over the micro-batches (iterations) of the
request.  Non-uniform t[m] (a full prompt next to decode-only micro-batches) is what creates the
bubbles (PB1-PB3); SARATHI's chunk + piggybacked decodes make t[m] nearly uniform.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


def pipeline_timeline(t: Sequence[float], stages: int) -> Tuple[List[List[float]], List[List[float]], List[float]]:
    """Returns (start[s][m], finish[s][m], bubble[m] = sum over stages of the idle time just
    before micro-batch m)."""
    if stages < 1:
        raise ValueError("stages >= 1")
    n = len(t)
    start = [[0.0] * n for _ in range(stages)]
    finish = [[0.0] * n for _ in range(stages)]
    bubble = [0.0] * n
    for m in range(n):
        for s in range(stages):
            ready = finish[s - 1][m] if s > 0 else (finish[stages - 1][m - stages] if m >= stages else 0.0)
            free = finish[s][m - 1] if m > 0 else 0.0
            start[s][m] = max(ready, free)
            finish[s][m] = start[s][m] + t[m]
            if m > 0:
                bubble[m] += start[s][m] - free
    return start, finish, bubble


def request_bubbles(micro_batches: Sequence[Sequence[int]], bubble: Sequence[float]) -> Dict[int, float]:
    """Per request: the sum of the bubbles of the micro-batches it took part in."""
    out: Dict[int, float] = {}
    for m, reqs in enumerate(micro_batches):
        for r in reqs:
            out[r] = out.get(r, 0.0) + bubble[m]
    return out

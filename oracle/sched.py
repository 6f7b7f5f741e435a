"""Reference scheduling, chunking and KV-slot arithmetic — TEST INFRASTRUCTURE ONLY.

Pure-integer Python; the C++ scheduler / block allocator in the library must match it
bit-exactly (north star: "bit-exactly on KV-cache slot indexing and scheduling").

Paper passages followed:
  * chunked-prefills: split a prompt of P tokens into chunks of C (§4.2); the
    remainder chunk is P-(N-1)C (reading O-14).
  * KV re-reads: "the first chunk's KV cache is loaded N times, the second ... N-1 times"
    (§4.2).
  * decode-maximal batching: "a single prefill chunk and piggybacking the remaining slots with
    decode tokens" (§4.3); at most B-1 decodes with a chunk, B without.
  * max batch size B = floor((M_G - M_S) / (L * m_kv)) (§4.3).
  * balanced P:D = C/(B-1) (§5.1.3); tile-adjusted chunk C-(B-1) (§4.4);
    chunk 128 at B=4 piggybacks P/128*3 ~ P/42 decodes (§4.4).
  * KV pre-allocated per max sequence length (§4.5) -> a request reserves
    ceil((P+D)/bs) blocks at admission, lowest-free-block-first (reading O-17);
    slot = table[pos // bs] * bs + pos % bs.
  * queue discipline FCFS by (arrival, id); all decode-phase requests ride along in admission
    order (reading O-16); a request's decodes never share a batch with its own chunk.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

# ---------------------------------------------------------------------------
# Chunking (§4.2) and the §4.3/§4.4/§5.1.3 formulas.
# ---------------------------------------------------------------------------


def plan_chunks(P: int, C: int) -> List[Tuple[int, int]]:
    """[(start, len)] tiling [0, P) with chunks of C; the last may be shorter (O-14)."""
    if P < 1 or C < 1:
        raise ValueError("P >= 1 and C >= 1 required")
    n = -(-P // C)
    return [(j * C, min(C, P - j * C)) for j in range(n)]


def chunk_key_ranges(start: int, length: int) -> List[Tuple[int, int]]:
    """Progressive causal mask of one chunk: query at global position q sees keys [0, q]."""
    return [(0, q) for q in range(start, start + length)]


def kv_reload_tokens(plan: Sequence[Tuple[int, int]]) -> int:
    """Token-KV reads over all chunks = sum_j (start_j + len_j)."""
    return sum(s + n for s, n in plan)


def max_batch_size(M_G: float, M_S: float, L: int, m_kv: float) -> int:
    """B = floor((M_G - M_S) / (L * m_kv)); 0 when nothing fits."""
    num = M_G - M_S
    if num <= 0:
        return 0
    return int(math.floor(num / (L * m_kv)))


def advise_chunk_size(C: int, B: int) -> int:
    """Tile-adjusted chunk C - (B-1) so chunk + (B-1) decodes = C."""
    if C <= B - 1:
        raise ValueError("chunk must exceed the decode count")
    return C - (B - 1)


def gemm_token_capacity(T: int) -> int:
    """Token columns the B200 swap-AB GEMM computes for T tokens (the padding is free): token tiles
    of <= 512; a tile of per <= 256 tokens is one UMMA of N = 16*ceil(per/16), a wider one two UMMAs
    with bn = 32*ceil(per/32) (the UMMA N quanta 16 / 32 of tcgen05.mma cta_group::2)."""
    T = max(T, 1)
    n_tiles = -(-T // 512)
    per = -(-T // n_tiles)
    bn = max(16, 16 * -(-per // 16)) if per <= 256 else 32 * -(-per // 32)
    return bn * n_tiles


def b200_chunk(C: int, d: int, remaining: int) -> int:
    """The paper's tile-quantization chunk rule (trim the chunk so chunk + decodes lands
    on the tile boundary) restated for the B200 GEMM's quanta (reading O-23): if
    T = C + d overshoots the cost step b = 512 (a second token tile) by at most C/8, trim to b - d;
    otherwise fill the padded tile to gemm_token_capacity(T) - d.  Clamped to [1, remaining]."""
    T = C + d
    p = gemm_token_capacity(T) - d
    for b in (512,):
        if b < T <= b + C // 8 and b - d >= 1:
            p = b - d
            break
    return max(1, min(p, remaining))


def optimal_pd(C: int, B: int) -> float:
    """Balanced P:D = C / (B-1)."""
    if B < 2:
        raise ValueError("B >= 2 required (no decode slots otherwise)")
    return C / (B - 1)


def piggyback_capacity(P: int, C: int, B: int) -> float:
    """Decodes that can ride along with one request's prefill: (P/C)(B-1)."""
    return P / C * (B - 1)


# ---------------------------------------------------------------------------
# KV block allocator and slot mapping (reading O-17).
# ---------------------------------------------------------------------------


class BlockAllocator:
    def __init__(self, num_blocks: int, block_size: int):
        if num_blocks < 0 or block_size < 1:
            raise ValueError("bad allocator geometry")
        self.num_blocks = num_blocks
        self.block_size = block_size
        self.free_set = set(range(num_blocks))
        self.tables: Dict[int, List[int]] = {}
        self.reserved: Dict[int, int] = {}

    def blocks_for(self, max_tokens: int) -> int:
        return -(-max_tokens // self.block_size)

    def can_alloc(self, max_tokens: int) -> bool:
        return self.blocks_for(max_tokens) <= len(self.free_set)

    def alloc(self, req_id: int, max_tokens: int) -> List[int]:
        if req_id in self.tables:
            raise ValueError("request already allocated")
        n = self.blocks_for(max_tokens)
        if n > len(self.free_set):
            raise MemoryError("not enough KV blocks")
        blocks = sorted(self.free_set)[:n]          # lowest-free-block-first
        for b in blocks:
            self.free_set.remove(b)
        self.tables[req_id] = blocks
        self.reserved[req_id] = max_tokens
        return list(blocks)

    def free(self, req_id: int) -> None:
        for b in self.tables.pop(req_id):
            self.free_set.add(b)
        self.reserved.pop(req_id)

    def slot(self, req_id: int, pos: int) -> int:
        return slot_of(self.tables[req_id], pos, self.block_size)


def slot_of(table: Sequence[int], pos: int, block_size: int) -> int:
    return table[pos // block_size] * block_size + pos % block_size


# ---------------------------------------------------------------------------
# Decode-maximal batching scheduler (§4.3) and the paper's comparison baselines (§5.1, §5.2).
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class ReqState:
    req_id: int
    P: int
    D: int
    arrival_iter: int
    prefill_done: int = 0
    decode_done: int = 0
    admitted: bool = False
    finished: bool = False
    admit_seq: int = -1


@dataclasses.dataclass
class Plan:
    iteration: int
    prefill: Optional[Tuple[int, int, int]]       # (req_id, start, n_tokens)
    decodes: List[Tuple[int, int]]                # [(req_id, position)]

    @property
    def num_tokens(self) -> int:
        return (self.prefill[2] if self.prefill else 0) + len(self.decodes)


SARATHI, REQUEST_LEVEL, ORCA_BEST = "sarathi", "request_level", "orca_best"


class Scheduler:
    """FCFS admission with up-front KV reservation; batch formation per policy.

    sarathi       : <= 1 chunk of min(C_eff, remaining) + decodes (<= B-1 with a chunk, else B)
    orca_best     : same with C = unbounded (one FULL prompt per batch, "special case of
                    Sarathi where the chunk size is set to the maximum sequence length")
    request_level : cohort of <= B requests; each prompt as its own prefill-only batch (the
                    C-ABI takes one prefill item per batch), then decode-only batches of the
                    cohort until it drains; no admission mid-cohort (P:L26 baseline)
    """

    def __init__(self, B: int, C: int, allocator: BlockAllocator, policy: str = SARATHI,
                 tile_adjust: int = 0):
        """tile_adjust: 0 the literal chunk C; 1 the paper's C - (B-1); 2 b200_chunk with
        the batch's own decode count."""
        if B < 1 or C < 1:
            raise ValueError("B >= 1 and C >= 1")
        self.B, self.C, self.alloc, self.policy = B, C, allocator, policy
        self.tile_adjust = tile_adjust
        self.reqs: Dict[int, ReqState] = {}
        self.iteration = 0
        self._admit_counter = 0

    def submit(self, req_id: int, P: int, D: int, arrival_iter: int = 0) -> None:
        if req_id in self.reqs or P < 1 or D < 0:
            raise ValueError("bad request")
        if self.alloc.blocks_for(P + D) > self.alloc.num_blocks:
            # never admissible: under strict FCFS it would block every later request (S: every
            # request eventually finishes; reading O-16)
            raise ValueError("P+D reservation exceeds the block pool")
        self.reqs[req_id] = ReqState(req_id, P, D, arrival_iter)

    def _running(self) -> List[ReqState]:
        return sorted((r for r in self.reqs.values() if r.admitted and not r.finished),
                      key=lambda r: r.admit_seq)

    def _pending(self) -> List[ReqState]:
        return sorted((r for r in self.reqs.values()
                       if not r.admitted and r.arrival_iter <= self.iteration),
                      key=lambda r: (r.arrival_iter, r.req_id))

    def _admit(self) -> None:
        if self.policy == REQUEST_LEVEL and self._running():
            return
        running = len(self._running())
        for r in self._pending():
            if running >= self.B or not self.alloc.can_alloc(r.P + r.D):
                break                               # strict FCFS: no skipping
            self.alloc.alloc(r.req_id, r.P + r.D)
            r.admitted, r.admit_seq = True, self._admit_counter
            self._admit_counter += 1
            running += 1

    def done(self) -> bool:
        return all(r.finished for r in self.reqs.values())

    def next_batch(self) -> Optional[Plan]:
        self._admit()
        running = self._running()
        prefill = None
        cand = [r for r in running if r.prefill_done < r.P]
        decoders = [r for r in running if r.prefill_done == r.P and r.decode_done < r.D]
        if self.policy == REQUEST_LEVEL:
            if cand:
                r = cand[0]
                prefill = (r.req_id, r.prefill_done, r.P - r.prefill_done)
                decoders = []
        elif cand:
            r = cand[0]
            rem = r.P - r.prefill_done
            if self.policy == ORCA_BEST:
                n = rem
            elif self.tile_adjust == 2:
                n = b200_chunk(self.C, min(len(decoders), self.B - 1), rem)
            else:
                n = min(advise_chunk_size(self.C, self.B) if self.tile_adjust == 1 else self.C, rem)
            prefill = (r.req_id, r.prefill_done, n)
        cap = self.B - 1 if prefill is not None else self.B
        decodes = [(r.req_id, r.P + r.decode_done) for r in decoders[:cap]]
        if prefill is None and not decodes:
            return None
        return Plan(self.iteration, prefill, decodes)

    def complete(self, plan: Plan) -> List[int]:
        """Advance state after a batch ran; returns the ids of requests that finished."""
        finished = []
        if plan.prefill is not None:
            r = self.reqs[plan.prefill[0]]
            r.prefill_done += plan.prefill[2]
            if r.prefill_done == r.P and r.D == 0:
                finished.append(r.req_id)
        for rid, _ in plan.decodes:
            r = self.reqs[rid]
            r.decode_done += 1
            if r.decode_done == r.D:
                finished.append(rid)
        for rid in finished:
            self.reqs[rid].finished = True
            self.alloc.free(rid)
        self.iteration += 1
        return finished

    def idle_step(self) -> None:
        self.iteration += 1


def run_schedule(sched: Scheduler, max_iters: int = 1 << 20) -> List[Plan]:
    plans = []
    while not sched.done():
        if len(plans) + 1 > max_iters:
            raise RuntimeError("schedule did not drain")
        p = sched.next_batch()
        if p is None:
            sched.idle_step()
            continue
        plans.append(p)
        sched.complete(p)
    return plans

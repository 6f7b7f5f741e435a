"""Thin ctypes binding of libsarathi.so (include/sarathi.h).

Argument marshalling only: every step of the hybrid-batch forward pass runs in the library's
CUDA kernels.  There is no fallback: if libsarathi.so is missing or fails to load, importing
the binding raises (build it with ``python -m paper_2308_16369_b200.build``).

Function names mirror the C ABI (``sarathi_init_model`` ...); ``Model`` and ``Scheduler`` are
convenience wrappers that hold the handles and convert Python/NumPy/torch arguments.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence, Tuple

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsarathi.so")

OK, EINVAL, ENOKV, EUNKNOWN_REQ, EDUP, EPOS, EOVERFLOW, ECUDA, ENCCL, ESTATE = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9
FFN_SWIGLU, FFN_GELU = 0, 1
RETURN_ALL_ROWS, DUMP_LAYERS, LOGITS_HOST, NO_LOGITS = 1, 2, 4, 8
POLICY_SARATHI, POLICY_ORCA_BEST, POLICY_REQUEST_LEVEL = 0, 1, 2
EPI_STORE_BF16, EPI_STORE_F32, EPI_ADD_F32, EPI_SILU_MUL, EPI_GELU = 0, 1, 2, 3, 4

# exported symbols (checked by the CPU test suite against include/sarathi.h)
EXPORTS = [
    "sarathi_nccl_unique_id", "sarathi_init_model", "sarathi_destroy", "sarathi_alloc_kv",
    "sarathi_kv_bytes_per_token", "sarathi_max_batch", "sarathi_request_alloc", "sarathi_request_free",
    "sarathi_request_cached_len", "sarathi_run_hybrid_batch", "sarathi_debug_slot_mapping",
    "sarathi_debug_block_table", "sarathi_debug_hidden", "sarathi_debug_kv", "sarathi_debug_weight",
    "sarathi_launch_count", "sarathi_last_error", "sarathi_sched_create", "sarathi_sched_destroy",
    "sarathi_sched_submit", "sarathi_sched_next", "sarathi_sched_complete", "sarathi_sched_idle_step",
    "sarathi_sched_done", "sarathi_sched_block_table", "sarathi_op_gemm", "sarathi_op_rmsnorm",
    "sarathi_request_truncate", "sarathi_last_io_bytes", "sarathi_set_profiling", "sarathi_op_times", "sarathi_op_kernel_times",
    "sarathi_op_pack_weight", "sarathi_shard_map", "sarathi_local_group_create", "sarathi_local_group_destroy",
    "sarathi_token_capacity", "sarathi_chunk_advice", "sarathi_stage_input", "sarathi_stage_output",
    "sarathi_chain_schedule",
]
GEMM_W_PACKED = 0x100
OP_NAMES = ["embed", "rmsnorm", "gemm_qkv", "prefill_attn", "decode_attn", "gemm_o", "gemm_gate_up",
            "gemm_down", "lm_head", "allreduce", "other", "gemm_chain"]


class SarathiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"sarathi error {code}: {msg}")
        self.code = code


class ModelConfigC(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_hidden", C.c_int32),
                ("vocab", C.c_int32), ("ffn_kind", C.c_int32), ("rms_eps", C.c_float),
                ("rope_base", C.c_float), ("max_seq_len", C.c_int32), ("max_tokens_per_batch", C.c_int32)]


class DistC(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("local_group", C.c_void_p),
                ("pp_stage", C.c_int32), ("pp_stages", C.c_int32)]


class PrefillChunkC(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("start_pos", C.c_int32), ("n_tokens", C.c_int32),
                ("token_ids", C.POINTER(C.c_int32))]


class DecodeSetC(C.Structure):
    _fields_ = [("n", C.c_int32), ("req_ids", C.POINTER(C.c_int64)), ("token_ids", C.POINTER(C.c_int32)),
                ("positions", C.POINTER(C.c_int32))]


class PlanC(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("prefill_req", C.c_int64), ("prefill_start", C.c_int32),
                ("prefill_len", C.c_int32), ("n_decodes", C.c_int32), ("n_admitted", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2308_16369_b200.build` (no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I32, I64, U64, VP, F = C.POINTER, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_float
    sig = {
        "sarathi_nccl_unique_id": [VP],
        "sarathi_init_model": [P(ModelConfigC), P(DistC), U64, P(VP), P(VP)],
        "sarathi_alloc_kv": [VP, I64, I32],
        "sarathi_kv_bytes_per_token": [VP, P(I64)],
        "sarathi_max_batch": [VP, I32, I64, P(I32)],
        "sarathi_request_alloc": [VP, I64, I32],
        "sarathi_request_free": [VP, I64],
        "sarathi_request_cached_len": [VP, I64, P(I32)],
        "sarathi_run_hybrid_batch": [VP, P(PrefillChunkC), P(DecodeSetC), VP, I32],
        "sarathi_debug_slot_mapping": [VP, P(I32), I32, P(I32)],
        "sarathi_debug_block_table": [VP, I64, P(I32), I32, P(I32)],
        "sarathi_debug_hidden": [VP, I32, P(F)],
        "sarathi_debug_kv": [VP, I32, I64, I32, I32, P(C.c_uint16), P(C.c_uint16)],
        "sarathi_debug_weight": [VP, I32, I32, I64, I64, P(C.c_uint16)],
        "sarathi_launch_count": [VP, P(I64)],
        "sarathi_sched_create": [I32, I32, I32, I32, I64, I32, P(VP)],
        "sarathi_sched_submit": [VP, I64, I32, I32, I32],
        "sarathi_sched_next": [VP, P(PlanC), P(I64), P(I32), P(I64), I32],
        "sarathi_sched_complete": [VP, P(I64), I32, P(I32)],
        "sarathi_sched_idle_step": [VP],
        "sarathi_sched_done": [VP, P(I32)],
        "sarathi_sched_block_table": [VP, I64, P(I32), I32, P(I32)],
        "sarathi_op_gemm": [VP, VP, VP, I32, I32, I32, I32, I32, VP],
        "sarathi_op_rmsnorm": [VP, VP, VP, I32, I32, F, VP],
        "sarathi_request_truncate": [VP, I64, I32],
        "sarathi_last_io_bytes": [VP, P(I64), P(I64)],
        "sarathi_set_profiling": [VP, I32],
        "sarathi_op_times": [VP, P(C.c_double), P(I64), I32, I32],
        "sarathi_op_kernel_times": [VP, P(C.c_double), P(I64), I32, I32],
        "sarathi_op_pack_weight": [VP, VP, I32, I32, VP],
        "sarathi_local_group_create": [I32, I32, P(VP)],
        "sarathi_token_capacity": [I32, P(I32), P(I32), P(I32)],
        "sarathi_chunk_advice": [I32, I32, I32, P(I32)],
        "sarathi_chain_schedule": [I32, P(I32), P(I32), P(I32), P(I32), P(C.c_double), I32, C.c_double, C.c_double,
                                   P(I32), P(I32), I32, P(I32), P(C.c_double)],
        "sarathi_stage_input": [VP, VP],
        "sarathi_stage_output": [VP, P(VP), P(I32)],
        "sarathi_shard_map": [P(ModelConfigC), I32, I32, I32, I32, P(I32), P(F), P(I64), I32, P(I32), P(I32)],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.sarathi_destroy.argtypes = [VP]
    lib.sarathi_destroy.restype = None
    lib.sarathi_local_group_destroy.argtypes = [VP]
    lib.sarathi_local_group_destroy.restype = None
    lib.sarathi_sched_destroy.argtypes = [VP]
    lib.sarathi_sched_destroy.restype = None
    lib.sarathi_last_error.argtypes = []
    lib.sarathi_last_error.restype = C.c_char_p
    return lib


lib = _load()


def _check(rc: int) -> int:
    if rc < 0:
        raise SarathiError(rc, lib.sarathi_last_error().decode(errors="replace"))
    return rc


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _p(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib.sarathi_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def config_from(cfg, max_tokens_per_batch: int, max_seq_len: Optional[int] = None) -> ModelConfigC:
    """Builds the C config from any object with the ModelConfig attribute names (e.g. synth)."""
    return ModelConfigC(cfg.n_layers, cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn_hidden,
                        cfg.vocab, cfg.ffn_kind, cfg.rms_eps, cfg.rope_base,
                        max_seq_len if max_seq_len is not None else cfg.max_seq_len, max_tokens_per_batch)


class Model:
    """Owns a sarathi_model handle (one per GPU / process)."""

    def __init__(self, cfg: ModelConfigC, seed: int, rank: int = 0, world: int = 1, device: int = 0,
                 nccl_id: Optional[bytes] = None, stream: int = 0,
                 host_tensors: Optional[Sequence[Optional[np.ndarray]]] = None,
                 local_group: Optional["LocalGroup"] = None, pp_stage: int = 0, pp_stages: int = 1):
        """host_tensors: None (weights generated on device from `seed`) or the 9*L + 3 logical bf16
        tensors (uint16 bit patterns, nn.Linear [out, in]) in the order of include/sarathi.h."""
        self.cfg = cfg
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        dist = DistC(rank, world, device, C.cast(self._idbuf, C.c_void_p) if self._idbuf else None,
                     C.c_void_p(stream) if stream else None, local_group.h if local_group is not None else None,
                     pp_stage, pp_stages)
        self._group = local_group  # keep the group alive while this handle exists
        ht = None
        if host_tensors is not None:
            if len(host_tensors) != 9 * cfg.n_layers + 3:
                raise ValueError(f"host_tensors: expected {9 * cfg.n_layers + 3} entries")
            keep = [None if t is None else np.ascontiguousarray(t, dtype=np.uint16) for t in host_tensors]
            ht = (C.c_void_p * len(keep))(*[None if t is None else t.ctypes.data for t in keep])
        h = C.c_void_p()
        _check(lib.sarathi_init_model(C.byref(cfg), C.byref(dist), C.c_uint64(seed), ht, C.byref(h)))
        self.h = h
        self.vocab = cfg.vocab

    def close(self):
        if getattr(self, "h", None):
            lib.sarathi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc_kv(self, num_blocks: int, block_size: int):
        _check(lib.sarathi_alloc_kv(self.h, num_blocks, block_size))

    def kv_bytes_per_token(self) -> int:
        v = C.c_int64()
        _check(lib.sarathi_kv_bytes_per_token(self.h, C.byref(v)))
        return v.value

    def max_batch(self, tokens_per_request: int, reserve_bytes: int = 0) -> int:
        v = C.c_int32()
        _check(lib.sarathi_max_batch(self.h, tokens_per_request, reserve_bytes, C.byref(v)))
        return v.value

    def request_alloc(self, req_id: int, max_tokens: int):
        _check(lib.sarathi_request_alloc(self.h, req_id, max_tokens))

    def request_free(self, req_id: int):
        _check(lib.sarathi_request_free(self.h, req_id))

    def cached_len(self, req_id: int) -> int:
        v = C.c_int32()
        _check(lib.sarathi_request_cached_len(self.h, req_id, C.byref(v)))
        return v.value

    def run_hybrid_batch(self, prefill: Optional[Tuple[int, int, Sequence[int]]],
                         decodes: Sequence[Tuple[int, int, int]], logits_ptr: int = 0, flags: int = 0,
                         logits_host: Optional[np.ndarray] = None) -> int:
        """prefill = (req_id, start_pos, tokens) or None; decodes = [(req_id, token, position)].

        logits_ptr: device pointer (fp32 [R][V]); or pass logits_host (fp32 numpy) to get a host copy.
        Returns R (rows written)."""
        keep = []
        pc = None
        p = 0
        if prefill is not None:
            rid, start, toks = prefill
            t = _i32(toks)
            keep.append(t)
            p = len(t)
            pc = PrefillChunkC(rid, start, p, _p(t, C.c_int32))
        d = len(decodes)
        ds = None
        if d:
            rq = _i64([x[0] for x in decodes])
            tk = _i32([x[1] for x in decodes])
            ps = _i32([x[2] for x in decodes])
            keep += [rq, tk, ps]
            ds = DecodeSetC(d, _p(rq, C.c_int64), _p(tk, C.c_int32), _p(ps, C.c_int32))
        ptr = logits_ptr
        R = (p + d) if flags & RETURN_ALL_ROWS else d + (1 if p else 0)
        if logits_host is not None:
            if logits_host.dtype != np.float32 or not logits_host.flags.c_contiguous:
                raise ValueError("logits_host must be a C-contiguous float32 array")
            if not flags & NO_LOGITS and logits_host.size < R * self.vocab:
                raise ValueError(f"logits_host holds {logits_host.size} floats < R*V = {R}*{self.vocab}")
            flags |= LOGITS_HOST
            ptr = logits_host.ctypes.data
        _check(lib.sarathi_run_hybrid_batch(self.h, C.byref(pc) if pc else None, C.byref(ds) if ds else None,
                                            C.c_void_p(ptr) if ptr else None, flags))
        return R

    def stage_input(self, h_ptr: int):
        """Pipeline stage > 0: device pointer (fp32 [T][H]) of the previous stage's output."""
        _check(lib.sarathi_stage_input(self.h, C.c_void_p(h_ptr)))

    def stage_output(self) -> Tuple[int, int]:
        """(device pointer of this stage's residual stream after its layers, T) for the last batch."""
        p, t = C.c_void_p(), C.c_int32()
        _check(lib.sarathi_stage_output(self.h, C.byref(p), C.byref(t)))
        return p.value, t.value

    def truncate(self, req_id: int, new_len: int):
        _check(lib.sarathi_request_truncate(self.h, req_id, new_len))

    def last_io_bytes(self) -> Tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        _check(lib.sarathi_last_io_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_profiling(self, on: bool):
        _check(lib.sarathi_set_profiling(self.h, int(on)))

    def op_times(self, reset: bool = True):
        """{op name: (total ms, launches)} accumulated since the last reset (syncs the stream)."""
        ms = np.zeros(len(OP_NAMES), dtype=np.float64)
        cnt = np.zeros(len(OP_NAMES), dtype=np.int64)
        _check(lib.sarathi_op_times(self.h, _p(ms, C.c_double), _p(cnt, C.c_int64), len(OP_NAMES), int(reset)))
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(OP_NAMES)}

    def op_kernel_times(self, reset: bool = True):
        """{op name: (total ms, launches)} of in-kernel device spans (GEMMs, decode and prefill attention)
        since the last reset."""
        ms = np.zeros(len(OP_NAMES), dtype=np.float64)
        cnt = np.zeros(len(OP_NAMES), dtype=np.int64)
        _check(lib.sarathi_op_kernel_times(self.h, _p(ms, C.c_double), _p(cnt, C.c_int64), len(OP_NAMES), int(reset)))
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(OP_NAMES)}

    def slot_mapping(self) -> np.ndarray:
        n = C.c_int32()
        _check(lib.sarathi_debug_slot_mapping(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(lib.sarathi_debug_slot_mapping(self.h, _p(out, C.c_int32), n.value, C.byref(n)))
        return out

    def block_table(self, req_id: int) -> np.ndarray:
        n = C.c_int32()
        _check(lib.sarathi_debug_block_table(self.h, req_id, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(lib.sarathi_debug_block_table(self.h, req_id, _p(out, C.c_int32), n.value, C.byref(n)))
        return out

    def hidden(self, layer: int, T: int) -> np.ndarray:
        out = np.zeros((T, self.cfg.hidden), dtype=np.float32)
        _check(lib.sarathi_debug_hidden(self.h, layer, _p(out, C.c_float)))
        return out

    def kv(self, layer: int, req_id: int, pos0: int, n: int, n_kv_local: int) -> Tuple[np.ndarray, np.ndarray]:
        k = np.zeros((n, n_kv_local, self.cfg.head_dim), dtype=np.uint16)
        v = np.zeros_like(k)
        _check(lib.sarathi_debug_kv(self.h, layer, req_id, pos0, n, _p(k, C.c_uint16), _p(v, C.c_uint16)))
        return k, v

    def weight(self, layer: int, tensor: int, offset: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint16)
        _check(lib.sarathi_debug_weight(self.h, layer, tensor, offset, count, _p(out, C.c_uint16)))
        return out

    def launch_count(self) -> int:
        v = C.c_int64()
        _check(lib.sarathi_launch_count(self.h, C.byref(v)))
        return v.value


class LocalGroup:
    """sarathi_local_group: `world` Model handles on one device, one host thread per rank (TP
    stand-in for one process per GPU; see include/sarathi.h)."""

    def __init__(self, world: int, device: int = 0):
        h = C.c_void_p()
        _check(lib.sarathi_local_group_create(world, device, C.byref(h)))
        self.h = h
        self.world = world

    def close(self):
        if getattr(self, "h", None):
            lib.sarathi_local_group_destroy(self.h)
            self.h = None


class Scheduler:
    """Host scheduler (decode-maximal batching, §4.3) — C++ implementation behind the C ABI."""

    def __init__(self, B: int, C_: int, num_blocks: int, block_size: int, policy: int = POLICY_SARATHI,
                 tile_adjust: int = 0):
        """tile_adjust: 0 literal chunk C, 1 the paper's C - (B-1), 2 the B200 advisor (chunk_advice)."""
        h = C.c_void_p()
        _check(lib.sarathi_sched_create(B, C_, policy, int(tile_adjust), num_blocks, block_size, C.byref(h)))
        self.h = h
        self.cap = max(B, 1) + 1024

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib.sarathi_sched_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def submit(self, req_id: int, P: int, D: int, arrival_iter: int = 0):
        _check(lib.sarathi_sched_submit(self.h, req_id, P, D, arrival_iter))

    def next(self):
        """Returns (plan or None, admitted ids).  plan = (prefill (req, start, n) | None, [(req, pos)])."""
        plan = PlanC()
        dr = np.zeros(self.cap, dtype=np.int64)
        dp = np.zeros(self.cap, dtype=np.int32)
        adm = np.zeros(self.cap, dtype=np.int64)
        have = _check(lib.sarathi_sched_next(self.h, C.byref(plan), _p(dr, C.c_int64), _p(dp, C.c_int32),
                                             _p(adm, C.c_int64), self.cap))
        admitted = [int(x) for x in adm[:plan.n_admitted]]
        if not have:
            return None, admitted
        pre = (int(plan.prefill_req), int(plan.prefill_start), int(plan.prefill_len)) if plan.prefill_req >= 0 else None
        decs = [(int(dr[i]), int(dp[i])) for i in range(plan.n_decodes)]
        return (pre, decs), admitted

    def complete(self):
        fin = np.zeros(self.cap, dtype=np.int64)
        n = C.c_int32()
        _check(lib.sarathi_sched_complete(self.h, _p(fin, C.c_int64), self.cap, C.byref(n)))
        return [int(x) for x in fin[:n.value]]

    def idle_step(self):
        _check(lib.sarathi_sched_idle_step(self.h))

    def done(self) -> bool:
        v = C.c_int32()
        _check(lib.sarathi_sched_done(self.h, C.byref(v)))
        return bool(v.value)

    def block_table(self, req_id: int) -> np.ndarray:
        n = C.c_int32()
        _check(lib.sarathi_sched_block_table(self.h, req_id, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(lib.sarathi_sched_block_table(self.h, req_id, _p(out, C.c_int32), n.value, C.byref(n)))
        return out


def token_capacity(T: int) -> Tuple[int, int, int]:
    """(capacity, n_tiles, n_mma) of the layer GEMMs' token tiling for a T-token batch (host only)."""
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib.sarathi_token_capacity(T, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def chunk_advice(C_: int, d: int, remaining: int) -> int:
    v = C.c_int32()
    _check(lib.sarathi_chunk_advice(C_, d, remaining, C.byref(v)))
    return v.value


def chain_schedule(jobs, pairs: int, e_add: float, e_fin: float):
    """Layer-chain work list (host only): jobs = [(pm_tiles, KB, split, dep_shift, e_done)].
    Returns (seg_off [pairs + 1], segs [n, 4] = (job, pair tile, kb0, kb1), predicted makespan)."""
    nj = len(jobs)
    col = lambda i, dt: np.ascontiguousarray([j[i] for j in jobs], dtype=dt)
    pm, kb, sp, ds, ed = col(0, np.int32), col(1, np.int32), col(2, np.int32), col(3, np.int32), col(4, np.float64)
    cap = 8 * pairs + 4 * int(sum(j[0] for j in jobs)) + 64
    off = np.zeros(pairs + 1, np.int32)
    segs = np.zeros(4 * cap, np.int32)
    n, ms = C.c_int32(), C.c_double()
    _check(lib.sarathi_chain_schedule(nj, _p(pm, C.c_int32), _p(kb, C.c_int32), _p(sp, C.c_int32), _p(ds, C.c_int32),
                                      _p(ed, C.c_double), pairs, e_add, e_fin, _p(off, C.c_int32), _p(segs, C.c_int32),
                                      cap, C.byref(n), C.byref(ms)))
    return off, segs[: 4 * n.value].reshape(-1, 4), ms.value


def op_gemm(W_ptr: int, X_ptr: int, out_ptr: int, M: int, N: int, K: int, mode: int, force_splits: int = 0,
            stream: int = 0):
    _check(lib.sarathi_op_gemm(C.c_void_p(W_ptr), C.c_void_p(X_ptr), C.c_void_p(out_ptr), M, N, K, mode,
                               force_splits, C.c_void_p(stream) if stream else None))


def op_pack_weight(W_ptr: int, out_ptr: int, rows: int, cols: int, stream: int = 0):
    _check(lib.sarathi_op_pack_weight(C.c_void_p(W_ptr), C.c_void_p(out_ptr), rows, cols,
                                      C.c_void_p(stream) if stream else None))


def shard_map(cfg: ModelConfigC, rank: int, world: int, layer: int, tensor: int):
    """(tau[rows], scale[rows], base[rows], (rows, cols)) of a rank's packed weight shard (host-only)."""
    rows, cols = C.c_int32(), C.c_int32()
    _check(lib.sarathi_shard_map(C.byref(cfg), rank, world, layer, tensor, None, None, None, 0, C.byref(rows),
                                 C.byref(cols)))
    tau = np.zeros(rows.value, np.int32)
    sc = np.zeros(rows.value, np.float32)
    base = np.zeros(rows.value, np.int64)
    _check(lib.sarathi_shard_map(C.byref(cfg), rank, world, layer, tensor, _p(tau, C.c_int32), _p(sc, C.c_float),
                                 _p(base, C.c_int64), rows.value, C.byref(rows), C.byref(cols)))
    return tau, sc, base, (rows.value, cols.value)


def op_rmsnorm(h_ptr: int, g_ptr: int, out_ptr: int, R: int, H: int, eps: float, stream: int = 0):
    _check(lib.sarathi_op_rmsnorm(C.c_void_p(h_ptr), C.c_void_p(g_ptr), C.c_void_p(out_ptr), R, H, eps,
                                  C.c_void_p(stream) if stream else None))

#!/usr/bin/env python
"""Benchmark of the SARATHI hybrid-batch forward pass on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]
    (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N; Megatron TP over NCCL)

A step = one decode-maximal hybrid batch (§4.3) of the headline composition through
sarathi_run_hybrid_batch: one prefill chunk of p = 256 tokens (chunk size 256) of a
1K prompt at cached prefix s = 768, plus d = 64 piggybacked decodes at context 1024 (LLaMA-13B,
BASELINE.json configs[1]).  All §8(a) rows run every step (embedding, 40 x [RMSNorm, QKV GEMM +
RoPE + KV append, chunked-prefill attention, paged decode attention, O GEMM + residual, RMSNorm,
gate/up GEMM + SiLU, down GEMM + residual], final norm + LM head on the R = d + 1 logit rows).
Requests are rolled back (sarathi_request_truncate) between steps so every step sees the same
composition.  Inputs are larger than L2 (26 GB of weights streamed per step).

value            hybrid-batch tokens/s = (p + d) / t_step, device-timed (CUDA events), max over ranks
marginal decode  (t(p=256,d) - t(p=256,d=0)) / d and the decode-only baseline
                 t(p=0,d)/d, timed the same way
e2e              same metric with host buffers through the public API: every step copies its
                 metadata (token ids, positions, slots, block tables) H2D and reads the logits D2H
roofline         dominant kernel (decode attention, HBM-bound) from per-op CUDA events
cpu_baseline     the fp64 oracle (oracle/) timed on this host's cores on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "hybrid-batch tokens/s & marginal decode ms/token, chunk=256, 1/2/4/8 B200 TP"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured"
        return d
    return dict(PEAKS_FALLBACK)


def ncu_traffic(kernel, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed ncu
    --set full capture of this workload (profiles/ncu_traffic.json, written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(workload, {}).get(kernel)
    return d


WORKLOADS = {
    # name: model, chunk p, prefix s, decodes d, decode context ctx (after append)
    "llama13b-p256-s768-d64-ctx1024": ("llama-13b", 256, 768, 64, 1024),
    "tiny-p16-s16-d3-ctx24": ("tiny", 16, 16, 3, 24),
}
DEFAULT_WORKLOAD = "llama13b-p256-s768-d64-ctx1024"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def setup_model(S, synth, cfg, p, s, d, ctx, rank, world, device, nccl_id, stream, block_size=64):
    max_tokens = 512
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=max_tokens), seed=0, rank=rank, world=world,
                device=device, nccl_id=nccl_id, stream=stream)
    n_req = d + 1
    per_req = max(s + p, ctx)
    blocks = n_req * -(-per_req // block_size) + 8
    m.alloc_kv(blocks, block_size)
    V = cfg.vocab
    tok = lambda r, a, n: synth.tokens(7, r, a, n, V)
    # request 0: the prefill request (cached prefix s); 1..d: decoders with ctx - 1 cached tokens
    m.request_alloc(0, s + p)
    for a in range(0, s, max_tokens):
        n = min(max_tokens, s - a)
        m.run_hybrid_batch((0, a, tok(0, a, n)), [], flags=S.NO_LOGITS)
    for r in range(1, d + 1):
        m.request_alloc(r, ctx)
        for a in range(0, ctx - 1, max_tokens):
            n = min(max_tokens, ctx - 1 - a)
            m.run_hybrid_batch((r, a, tok(r, a, n)), [], flags=S.NO_LOGITS)
    prefill = (0, s, tok(0, s, p))
    decodes = [(r, int(tok(r, ctx - 1, 1)[0]), ctx - 1) for r in range(1, d + 1)]
    return m, prefill, decodes


def ours(args):
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    model_name, p, s, d, ctx = WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    m, prefill, decodes = setup_model(S, synth, cfg, p, s, d, ctx, rank, world, local, nccl_id, sh)
    R = d + 1
    logits = torch.empty((R, cfg.vocab), dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def step(pre, decs, flags=0, host_out=None):
        if pre is not None:
            m.truncate(pre[0], pre[1])
        for r, _, pos in decs:
            m.truncate(r, pos)
        return m.run_hybrid_batch(pre, decs, logits_ptr=logits.data_ptr() if host_out is None else 0,
                                  flags=flags, logits_host=host_out)

    def timed(pre, decs, K, W):
        for _ in range(W):
            step(pre, decs)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        prof = os.environ.get("SARATHI_PROFILE_TIMED") == "1" and pre is not None and len(decs) > 0
        if prof:  # ncu --profile-from-start off captures exactly the timed hybrid steps
            torch.cuda.profiler.start()
        e0.record(stream)
        for _ in range(K):
            step(pre, decs)
        e1.record(stream)
        e1.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        barrier()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / K

    clocks = ClockSampler(local)
    launches0 = m.launch_count()
    clocks.start()
    ms_hybrid = timed(prefill, decodes, args.steps, args.warmup)
    clk = clocks.stop()
    launches = (m.launch_count() - launches0) // (args.steps + args.warmup)
    ms_prefill_only = timed(prefill, [], args.steps, max(1, args.warmup // 2))
    ms_decode_only = timed(None, decodes, args.steps, max(1, args.warmup // 2))
    # per-op CUDA-event timers over a separate profiled pass of the same composition
    m.set_profiling(True)
    m.op_times(reset=True)
    for _ in range(args.steps):
        step(prefill, decodes)
    ops = m.op_times(reset=True)
    kops = m.op_kernel_times(reset=True)  # in-kernel device spans of the same GEMM launches
    # the same decodes without the chunk: decode attention alone on the GPU (in the hybrid step the
    # chunked-prefill attention runs concurrently with it and shares the SMs)
    for _ in range(args.steps):
        step(None, decodes)
    ops_dec = m.op_times(reset=True)
    kops_dec = m.op_kernel_times(reset=True)
    m.set_profiling(False)
    # e2e: host buffers through the public API (H2D metadata + D2H logits every step), wall clock
    host_logits = np.empty((R, cfg.vocab), dtype=np.float32)
    host_logits_pinned = torch.empty((R, cfg.vocab), dtype=torch.float32).pin_memory()
    hl = host_logits_pinned.numpy()
    for _ in range(2):
        step(prefill, decodes, host_out=hl)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(prefill, decodes, host_out=hl)
    t1 = time.perf_counter()
    e2e_ms = (t1 - t0) * 1e3 / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d, d2h = m.last_io_bytes()
    del host_logits

    T = p + d
    value = T / (ms_hybrid / 1e3)
    peaks = load_peaks()
    # roofline of the dominant kernel: decode attention (HBM).  Algorithmic bytes per launch
    # = sum_j ctx_j * 2 (K,V) * n_kv_local * hd * 2 B, one launch per layer.
    nkv_l = cfg.n_kv_heads // world
    da_ms, da_n = ops["decode_attn"]
    da_bytes = d * ctx * 2 * nkv_l * cfg.head_dim * 2
    da_avg_s = (da_ms / max(da_n, 1)) / 1e3
    da_gbs = da_bytes / da_avg_s / 1e9 if da_avg_s > 0 else 0.0
    dd_ms, dd_n = ops_dec["decode_attn"]
    dd_avg_s = (dd_ms / max(dd_n, 1)) / 1e3
    dd_gbs = da_bytes / dd_avg_s / 1e9 if dd_avg_s > 0 else 0.0
    # GEMM tensor roofline (all four layer GEMMs, algorithmic 2*T*W flops)
    H, H2 = cfg.hidden, cfg.ffn_hidden
    ffn_mats = 3 if cfg.ffn_kind == synth.FFN_SWIGLU else 2
    w = {"gemm_qkv": (cfg.q_dim + 2 * cfg.kv_dim) * H, "gemm_o": cfg.q_dim * H,
         "gemm_gate_up": (ffn_mats - 1) * H2 * H, "gemm_down": H2 * H}
    gemm = {}
    for k, params in w.items():
        t_ms, n = ops[k]
        flops = 2.0 * T * params / world
        byts = 2.0 * params / world
        avg = t_ms / max(n, 1) / 1e3
        # GEMMs run inside a long step at the power-limited clock: the contract's peak for them is
        # the SUSTAINED measured bf16 figure; the burst fraction is reported beside it
        sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        gemm[k] = {"us": round(avg * 1e6, 2), "tflops": round(flops / avg / 1e12, 1) if avg else 0,
                   "weight_gbs": round(byts / avg / 1e9, 1) if avg else 0,
                   "frac_tensor": round(flops / avg / 1e12 / sus, 3) if avg else 0,
                   "frac_tensor_burst": round(flops / avg / 1e12 / peaks["bf16_tflops"], 3) if avg else 0}
        # the event-timed figure above includes launch gaps and event overhead of the profiled pass;
        # the kernel's own device span (first CTA start -> last CTA end, globaltimer) beside it
        kt_ms, kn = kops.get(k, (0.0, 0))
        if kn:
            kavg = kt_ms / kn / 1e3
            gemm[k]["us_kernel"] = round(kavg * 1e6, 2)
            gemm[k]["frac_tensor_kernel"] = round(flops / kavg / 1e12 / sus, 3)
    per_layer_ops = {k: {"ms_total": round(v[0], 3), "launches": v[1]} for k, v in ops.items() if v[1]}
    # device spans (first CTA start after its grid dependency -> last CTA end, globaltimer) of the
    # attention kernels: CUDA events on a stream running beside another grid are stamped late
    def span_us(kd, k):
        t_ms, n = kd.get(k, (0.0, 0))
        return round(t_ms / n * 1e3, 2) if n else None
    traffic = ncu_traffic("decode_attention", args.workload)
    roofline = {"kernel": "decode_attention", "bound": "hbm", "achieved": round(da_gbs, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(da_gbs / peaks["hbm_gbs"], 3),
                "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None,
                "algorithmic_bytes_per_launch": da_bytes,
                "avg_launch_us": round(da_avg_s * 1e6, 2), "peak_source": peaks["source"],
                "note": "hybrid step: the chunk's prefill attention runs concurrently (attention chain)",
                "span_us": span_us(kops, "decode_attn"),
                "prefill_attn_span_us": span_us(kops, "prefill_attn"),
                "alone": {"achieved": round(dd_gbs, 1), "frac": round(dd_gbs / peaks["hbm_gbs"], 3),
                          "avg_launch_us": round(dd_avg_s * 1e6, 2), "span_us": span_us(kops_dec, "decode_attn"),
                          "pass": "decode-only steps of the same decodes (no concurrent kernel)"}}

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_hybrid, 4),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (counter-based generator weights/tokens, seed 0)",
        "config": {"workload": args.workload, "model_shape": model_name, "p": p, "s": s, "d": d, "ctx": ctx,
                   "chunk": 256, "T": T, "parallelism": f"tp{world}", "kv_block_size": 64,
                   "l2": "inputs larger than L2 (all layer weights streamed every step)"},
        "marginal_decode_ms_per_token": round((ms_hybrid - ms_prefill_only) / d, 5),
        "decode_only_ms_per_token": round(ms_decode_only / d, 5),
        "decode_speedup": round((ms_decode_only / d) / max((ms_hybrid - ms_prefill_only) / d, 1e-9), 2),
        "prefill_only_ms": round(ms_prefill_only, 4), "decode_only_ms": round(ms_decode_only, 4),
        "e2e": {"value": round(T / (e2e_ms / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)},
        "roofline": roofline,
        "gemm_roofline": gemm,
        "op_breakdown_ms_over_steps": per_layer_ops,
        "gpu_launches": int(launches) * args.steps,
        "gpu_launches_per_step": int(launches),
        "clocks": clk,
    }
    if rank == 0:
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, p, s, d, ctx, budget_s=args.cpu_budget)
        print(json.dumps(out), flush=True)
    m.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# fp64 oracle on host cores (cpu_baseline leg and the --impl reference arm)
# ---------------------------------------------------------------------------
def _oracle_sample(cfg, p, s, d, ctx, n_pre=8, n_dec=8):
    """Bounded sample of the workload for the fp64 oracle: one full-width layer for n_pre chunk rows
    (prefix s + i) and n_dec decode rows (context ctx), with synthetic KV contexts of the right shape."""
    import synth
    from oracle import model as om
    lw = om.layer_weights(cfg, 0, 0)
    rng = np.random.default_rng(0)
    rows_pos = [s + p - n_pre + i for i in range(n_pre)] + [ctx - 1] * n_dec
    h_in = rng.standard_normal((len(rows_pos), cfg.hidden))
    kc = [rng.standard_normal((ps + 1, cfg.n_kv_heads, cfg.head_dim)) for ps in rows_pos]
    vc = [rng.standard_normal((ps + 1, cfg.n_kv_heads, cfg.head_dim)) for ps in rows_pos]
    wlm = synth.as_f64(synth.lm_head_rows_bits(cfg, 0, range(0, cfg.vocab, max(1, cfg.vocab // 2048))))
    gf = synth.as_f64(synth.final_gain_bits(cfg, 0))
    return lw, np.array(rows_pos), h_in, kc, vc, wlm, gf


def _oracle_time(cfg, sample, reps_budget_s):
    from oracle import model as om
    lw, pos, h_in, kc, vc, wlm, gf = sample
    t_layer = []
    t0 = time.perf_counter()
    while True:
        a = time.perf_counter()
        h = om.layer_rows_from_input(cfg, lw, h_in, pos, kc, vc)
        t_layer.append(time.perf_counter() - a)
        if time.perf_counter() - t0 > reps_budget_s:
            break
    a = time.perf_counter()
    om.logits_rows(cfg, gf, wlm, h)
    t_head = (time.perf_counter() - a) * (cfg.vocab / wlm.shape[0])
    layer = min(t_layer)
    proj = layer * cfg.n_layers + t_head
    return len(pos) / proj, layer, t_head


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return os.cpu_count()


def cpu_baseline(cfg, p, s, d, ctx, budget_s=10.0):
    t0 = time.perf_counter()
    sample = _oracle_sample(cfg, p, s, d, ctx)
    gen_s = time.perf_counter() - t0
    tps, layer_s, head_s = _oracle_time(cfg, sample, budget_s)
    n = len(sample[1])
    return {"value": round(tps, 3), "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
            "sample": (f"one full-width {cfg.name} layer (fp64 NumPy oracle) for {n} hybrid-batch rows "
                       f"(8 chunk rows at prefix ~{s + p}, 8 decode rows at ctx {ctx}) best of repeats, "
                       f"projected x{cfg.n_layers} layers + LM head; layer {layer_s:.3f}s, head {head_s:.3f}s; "
                       f"weight regeneration {gen_s:.1f}s excluded"),
            "host_cpu_count": os.cpu_count()}


def reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    model_name, p, s, d, ctx = WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    sample = _oracle_sample(cfg, p, s, d, ctx)
    per_step_budget = max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        _oracle_time(cfg, sample, 0.0)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tps, layer_s, head_s = _oracle_time(cfg, sample, 0.0)
        vals.append(tps)
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    n = len(sample[1])
    out = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall * 1e3 / max(args.steps, 1), 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, "model_shape": model_name, "p": p, "s": s,
                                          "d": d, "ctx": ctx, "chunk": 256, "T": p + d},
        "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
                         "sample": f"per step: one full-width {cfg.name} layer for {n} rows, projected to "
                                   f"{cfg.n_layers} layers + LM head (fp64 NumPy oracle)"},
        "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    _ = per_step_budget


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()

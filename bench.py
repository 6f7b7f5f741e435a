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
    # fixed compositions — name: model, chunk p, prefix s, decodes d, decode context ctx (after append)
    "llama13b-p256-s768-d64-ctx1024": ("llama-13b", 256, 768, 64, 1024),
    "tiny-p16-s16-d3-ctx24": ("tiny", 16, 16, 3, 24),
}
# request workloads driven through the C++ scheduler (sarathi_sched_*): PAPER.md L10-11 (§5.3) —
# lengths ~ Zipf(theta = 0.4) over [1K, 4K], P:D = 10, chunk 256, batch B = 27 (SURVEY §8(d)
# configs 4/5 generator; at N GPUs the model runs TP = N, the TP-scaling row of §8(d))
ZIPF_WORKLOADS = {
    # name: model, requests, B, C, P:D, workload seed
    "zipf-p10-llama13b": ("llama-13b", 64, 27, 256, 10.0, 4),
    "zipf-p10-tiny": ("tiny", 12, 4, 16, 10.0, 4),
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
def setup_model(S, synth, cfg, p, s, d, ctx, rank, world, device, nccl_id, stream, block_size=64, max_tokens=512):
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


def _dist_setup(args, S):
    import torch
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
    return rank, world, local, dist, nccl_id


def _max_over_ranks(dist, x):
    import torch
    if dist is None:
        return x
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


REPEATS = 3  # timed regions of the hybrid step and the e2e pass, interleaved; medians reported


def ours(args):
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    if args.workload in ZIPF_WORKLOADS:
        return ours_zipf(args)
    rank, world, local, dist, nccl_id = _dist_setup(args, S)
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    model_name, p, s, d, ctx = WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    table = model_name == "llama-13b"  # Table tbl-compute-split replica (T up to 1024)
    m, prefill, decodes = setup_model(S, synth, cfg, p, s, d, ctx, rank, world, local, nccl_id, sh,
                                      max_tokens=1024 if table else 512)
    R = d + 1
    logits = torch.empty((max(R, 8), cfg.vocab), dtype=torch.float32, device="cuda")

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
        """W untimed steps, then EXACTLY K steps between barrier + synchronize, CUDA events on the
        library stream; max over ranks."""
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
        return _max_over_ranks(dist, e0.elapsed_time(e1)) / K

    # e2e: host buffers through the public API (H2D metadata + D2H logits + sync every step), wall clock
    host_logits_pinned = torch.empty((R, cfg.vocab), dtype=torch.float32).pin_memory()
    hl = host_logits_pinned.numpy()

    def e2e_pass(K):
        for _ in range(2):
            step(prefill, decodes, host_out=hl)
        barrier()
        t0 = time.perf_counter()
        for _ in range(K):
            step(prefill, decodes, host_out=hl)
        t1 = time.perf_counter()
        return _max_over_ranks(dist, (t1 - t0) * 1e3 / K)

    clocks = ClockSampler(local)
    launches0 = m.launch_count()
    hyb, e2e = [], []
    clocks.start()
    for rep in range(REPEATS):
        hyb.append(timed(prefill, decodes, args.steps, args.warmup if rep == 0 else 2))
        e2e.append(e2e_pass(args.steps))
    clk = clocks.stop()
    launches = m.launch_count() - launches0
    ms_hybrid = statistics.median(hyb)
    e2e_ms = statistics.median(e2e)
    h2d, d2h = m.last_io_bytes()
    # launches per step from one extra counted step
    l0 = m.launch_count()
    step(prefill, decodes)
    launches_per_step = m.launch_count() - l0
    barrier()
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

    # Table tbl-compute-split replica (LLaMA-13B): prefill-only 1024 tokens,
    # decode-only d = 4 at sequence length 1024, mixed 1021-token prefill + 3 decodes
    tbl = None
    if table and d >= 4:
        tok = lambda r, a, n: synth.tokens(7, r, a, n, cfg.vocab)
        pre1024 = (0, 0, tok(0, 0, 1024))
        pre1021 = (0, 0, tok(0, 0, 1021))
        t_pre = timed(pre1024, [], args.steps, 2)
        t_pre1021 = timed(pre1021, [], args.steps, 2)
        t_dec = timed(None, decodes[:4], args.steps, 2)
        t_mix = timed(pre1021, decodes[:3], args.steps, 2)
        tbl = {"prefill_only_1024_ms": round(t_pre, 4), "decode_only_d4_ctx1024_ms": round(t_dec, 4),
               "mixed_1021p_3d_ms": round(t_mix, 4), "prefill_only_1021_ms": round(t_pre1021, 4),
               "per_token_prefill_ms": round(t_pre / 1024, 5),
               "decode_only_per_token_ms": round(t_dec / 4, 4),
               "marginal_decode_ms_paper_formula": round((t_mix - t_pre) / 3, 4),
               "marginal_decode_ms_vs_prefill_1021": round((t_mix - t_pre1021) / 3, 4),
               "decode_speedup": round((t_dec / 4) / max((t_mix - t_pre1021) / 3, 1e-9), 2),
               "paper_a6000_ms": {"prefill_only": 234.8, "decode_only": 49.96, "mixed": 238.4,
                                  "per_token_decode_only": 12.49, "marginal": 1.2},
               "note": "marginal_decode_ms_paper_formula = (mixed - prefill_only_1024)/3 as P:L421-423 "
                       "(the mixed batch has 3 fewer prefill tokens, so it can go negative when linears are "
                       "tensor-bound); the vs_prefill_1021 figure subtracts the same chunk"}

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
    gemm = gemm_roofline(cfg, synth, world, T, ops, kops, peaks)
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

    # the dominant kernel of the step: the layer chain (one launch per layer of O + FFN1 + FFN2 +
    # next QKV, tensor-bound) when its per-launch time exceeds the decode attention's, else the
    # decode attention; the other one is reported beside it (roofline_secondary)
    ch = gemm.get("gemm_chain")
    if ch and ch["us"] > da_avg_s * 1e6:
        sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        ctraffic = ncu_traffic("gemm_chain", args.workload)
        roofline_chain = {"kernel": "gemm_chain", "bound": "tensor", "achieved": ch["tflops"], "peak": sus,
                          "unit": "TFLOP/s", "frac": ch["frac_tensor"],
                          "traffic": ctraffic["dram_bytes_per_launch"] if ctraffic else None,
                          "traffic_source": ctraffic["source"] if ctraffic else None,
                          "algorithmic_flops_per_launch": round(ch["tflops"] * 1e12 * ch["us"] * 1e-6),
                          "avg_launch_us": ch["us"], "span_us": ch.get("us_kernel"),
                          "frac_span": ch.get("frac_tensor_kernel"), "frac_burst": ch["frac_tensor_burst"],
                          "peak_source": peaks["source"] + " (sustained bf16: the chain runs at the power-capped clock)",
                          "note": "per-op CUDA events of the profiled pass; span = first CTA past its grid "
                                  "dependency -> last CTA end"}
        roofline, roofline_secondary = roofline_chain, roofline
    else:
        # gemm_bf16_pair over the four layer GEMMs (QKV, O, gate||up, down): the kernel function
        # with the largest share of the step in the ncu launch list (~58 % vs the decode attention's
        # ~32 %); per-layer figures (four launches), tensor-bound against the sustained bf16 peak
        lay = gemm.get("all_layer_gemms")
        if lay and lay.get("us"):
            sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
            lay_fl = lay["frac_tensor"] * sus * 1e12 * lay["us"] * 1e-6
            gtraffic = ncu_traffic("gemm_layer", args.workload)
            roofline_gemm = {"kernel": "gemm_bf16_pair (QKV + O + gate_up + down of one layer)", "bound": "tensor",
                             "achieved": round(lay_fl / (lay["us"] * 1e-6) / 1e12, 1), "peak": sus,
                             "unit": "TFLOP/s", "frac": lay["frac_tensor"],
                             "traffic": gtraffic["dram_bytes_per_launch"] if gtraffic else None,
                             "traffic_source": gtraffic["source"] if gtraffic else None,
                             "traffic_unit": "bytes per layer (4 launches)",
                             "algorithmic_flops_per_layer": round(lay_fl),
                             "algorithmic_weight_bytes_per_layer": round(sum(
                                 v["weight_gbs"] * 1e9 * v["us"] * 1e-6 for k, v in gemm.items() if k.startswith("gemm_"))),
                             "us_per_layer": lay["us"], "frac_span": lay.get("frac_tensor_kernel"),
                             "peak_source": peaks["source"] + " (sustained bf16: the GEMMs run at the power-capped clock)",
                             "note": "per-op CUDA events of the profiled pass (they break the PDL chain: launch gaps "
                                     "included); frac_span = the kernels' own device spans"}
            roofline, roofline_secondary = roofline_gemm, roofline
        else:
            roofline_secondary = None

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_hybrid, 4),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (counter-based generator weights/tokens, seed 0)",
        "config": {"workload": args.workload, "model_shape": model_name, "p": p, "s": s, "d": d, "ctx": ctx,
                   "chunk": 256, "T": T, "parallelism": f"tp{world}", "kv_block_size": 64,
                   "l2": "inputs larger than L2 (all layer weights streamed every step)"},
        "repeats": {"n": REPEATS, "hybrid_ms_per_step": [round(x, 4) for x in hyb],
                    "e2e_ms_per_step": [round(x, 4) for x in e2e],
                    "how": f"{REPEATS} timed regions of exactly {args.steps} hybrid steps, each followed by an "
                           f"e2e pass of {args.steps} steps (interleaved); value / e2e = medians"},
        "marginal_decode_ms_per_token": round((ms_hybrid - ms_prefill_only) / d, 5),
        "decode_only_ms_per_token": round(ms_decode_only / d, 5),
        "decode_speedup": round((ms_decode_only / d) / max((ms_hybrid - ms_prefill_only) / d, 1e-9), 2),
        "prefill_only_ms": round(ms_prefill_only, 4), "decode_only_ms": round(ms_decode_only, 4),
        "e2e": {"value": round(T / (e2e_ms / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)},
        "roofline": roofline,
        "roofline_secondary": roofline_secondary,
        "gemm_roofline": gemm,
        "op_breakdown_ms_over_steps": per_layer_ops,
        "gpu_launches": int(launches_per_step) * args.steps,
        "gpu_launches_per_step": int(launches_per_step),
        "clocks": clk,
    }
    if tbl:
        out["tbl_compute_split"] = tbl
    _ = launches
    if rank == 0:
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, p, s, d, ctx, budget_s=args.cpu_budget)
        print(json.dumps(out), flush=True)
    m.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def gemm_roofline(cfg, synth, world, T, ops, kops, peaks):
    """Tensor roofline of the four layer GEMMs (algorithmic 2*T*W/t flops per launch)."""
    H, H2 = cfg.hidden, cfg.ffn_hidden
    ffn_mats = 3 if cfg.ffn_kind == synth.FFN_SWIGLU else 2
    w = {"gemm_qkv": (cfg.q_dim + 2 * cfg.kv_dim) * H, "gemm_o": cfg.q_dim * H,
         "gemm_gate_up": (ffn_mats - 1) * H2 * H, "gemm_down": H2 * H}
    gemm = {}
    sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    tot_flops, tot_s, tot_ks = 0.0, 0.0, 0.0
    for k, params in w.items():
        t_ms, n = ops[k]
        if n == 0:
            continue
        flops = 2.0 * T * params / world
        byts = 2.0 * params / world
        avg = t_ms / max(n, 1) / 1e3
        # GEMMs run inside a long step at the power-limited clock: the contract's peak for them is
        # the SUSTAINED measured bf16 figure; the burst fraction is reported beside it
        gemm[k] = {"us": round(avg * 1e6, 2), "tflops": round(flops / avg / 1e12, 1) if avg else 0,
                   "weight_gbs": round(byts / avg / 1e9, 1) if avg else 0,
                   "frac_tensor": round(flops / avg / 1e12 / sus, 3) if avg else 0,
                   "frac_tensor_burst": round(flops / avg / 1e12 / peaks["bf16_tflops"], 3) if avg else 0}
        tot_flops += flops
        tot_s += avg
        # the event-timed figure above includes launch gaps and event overhead of the profiled pass;
        # the kernel's own device span (first CTA start -> last CTA end, globaltimer) beside it
        kt_ms, kn = kops.get(k, (0.0, 0))
        if kn:
            kavg = kt_ms / kn / 1e3
            tot_ks += kavg
            gemm[k]["us_kernel"] = round(kavg * 1e6, 2)
            gemm[k]["frac_tensor_kernel"] = round(flops / kavg / 1e12 / sus, 3)
    # layer chain (gemm_chain.cu): one launch per layer = O + FFN1 + FFN2 (+ the next layer's QKV
    # for every layer but the last); the standalone launches above are then layer 0's QKV only
    c_ms, cn = ops.get("gemm_chain", (0.0, 0))
    if cn:
        L = cfg.n_layers
        steps = cn / L
        qkv_fl = 2.0 * T * w["gemm_qkv"] / world
        rest_fl = sum(2.0 * T * w[k] / world for k in ("gemm_o", "gemm_gate_up", "gemm_down"))
        fl = (L * rest_fl + (L - 1) * qkv_fl) / L  # per launch
        avg = c_ms / cn / 1e3
        ent = {"us": round(avg * 1e6, 2), "launches_per_step": L, "tflops": round(fl / avg / 1e12, 1),
               "frac_tensor": round(fl / avg / 1e12 / sus, 3),
               "frac_tensor_burst": round(fl / avg / 1e12 / peaks["bf16_tflops"], 3),
               "gemms": "O + FFN1 + FFN2 + next layer's QKV (RMSNorm folded in)"}
        kt_ms, kn = kops.get("gemm_chain", (0.0, 0))
        if kn:
            kavg = kt_ms / kn / 1e3
            ent["us_kernel"] = round(kavg * 1e6, 2)
            ent["frac_tensor_kernel"] = round(fl / kavg / 1e12 / sus, 3)
        gemm["gemm_chain"] = ent
        # per layer: the chain's share plus layer 0's standalone QKV amortised over the layers
        q_ms, qn = ops.get("gemm_qkv", (0.0, 0))
        lay_s = (c_ms + q_ms) / 1e3 / (steps * L)
        lay_fl = rest_fl + qkv_fl
        gemm["all_layer_gemms"] = {"us": round(lay_s * 1e6, 2), "frac_tensor": round(lay_fl / lay_s / 1e12 / sus, 3)}
        if kn:
            qk_ms, qkn = kops.get("gemm_qkv", (0.0, 0))
            lay_ks = (kt_ms + qk_ms) / 1e3 / (steps * L)
            gemm["all_layer_gemms"]["frac_tensor_kernel"] = round(lay_fl / lay_ks / 1e12 / sus, 3)
        return gemm
    if tot_s > 0:
        gemm["all_layer_gemms"] = {"us": round(tot_s * 1e6, 2), "frac_tensor": round(tot_flops / tot_s / 1e12 / sus, 3),
                                   "frac_tensor_kernel": round(tot_flops / tot_ks / 1e12 / sus, 3) if tot_ks else None}
    return gemm


def ours_zipf(args):
    """Request workload through the C++ scheduler (decode-maximal batching, C = 256, <= B-1
    piggybacked decodes): all requests arrive at t = 0; one step = one scheduler iteration
    (one run_hybrid_batch).  value = sum over iterations of (p + d) / device time of the whole run
    (CUDA events, max over ranks: hybrid-batch tokens/s aggregated over the workload's
    compositions); e2e = sum_r (P_r + D_r) / wall-clock makespan of a second run in which every
    iteration copies its metadata H2D and reads its logits D2H (a serving loop)."""
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    rank, world, local, dist, nccl_id = _dist_setup(args, S)
    model_name, n_req, B, C, pd, wseed = ZIPF_WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    lo, hi = (1024, 4096) if model_name != "tiny" else (24, 96)
    reqs = synth.zipf_workload(wseed, n_req, pd, lo=lo, hi=hi)
    stream = torch.cuda.Stream()
    bs = 64 if model_name != "tiny" else 16
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=C + B, max_seq_len=hi), seed=0, rank=rank, world=world,
                device=local, nccl_id=nccl_id, stream=stream.cuda_stream)
    num_blocks = B * -(-hi // bs) + 8
    m.alloc_kv(num_blocks, bs)
    logits = torch.empty((B + 1, cfg.vocab), dtype=torch.float32, device="cuda")
    hl = torch.empty((B + 1, cfg.vocab), dtype=torch.float32).pin_memory().numpy()
    V = cfg.vocab

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def run(specs, host, id_base):
        sched = S.Scheduler(B, C, num_blocks, bs)
        PD = {}
        for r in specs:
            sched.submit(id_base + r.req_id, r.prompt_len, r.decode_len, 0)
            PD[id_base + r.req_id] = (r.prompt_len, r.decode_len)
        iters, toks = 0, 0
        comp = []
        io = [0, 0]
        while not sched.done():
            plan, admitted = sched.next()
            for rid in admitted:
                m.request_alloc(rid, sum(PD[rid]))
            if plan is None:
                sched.idle_step()
                continue
            pre, decs = plan
            tk = lambda r, a, n=1: synth.tokens(11, r, a, n, V)
            prefill = (pre[0], pre[1], tk(pre[0], pre[1], pre[2])) if pre is not None else None
            dd = [(rid, int(tk(rid, pos)[0]), pos) for rid, pos in decs]
            if host:
                m.run_hybrid_batch(prefill, dd, logits_host=hl)
                a_, b_ = m.last_io_bytes()
                io[0] += a_
                io[1] += b_
            else:
                m.run_hybrid_batch(prefill, dd, logits_ptr=logits.data_ptr())
            iters += 1
            toks += (pre[2] if pre else 0) + len(decs)
            comp.append(((pre[2] if pre else 0), len(decs)))
            for rid in sched.complete():
                m.request_free(rid)
        return iters, toks, comp, io

    # warm-up: the first W requests' worth of iterations on a small sub-workload
    warm = synth.zipf_workload(wseed + 100, max(2, args.warmup), pd, lo=lo, hi=hi)
    run(warm, False, 1 << 40)
    run(warm, True, 1 << 39)
    clocks = ClockSampler(local)
    barrier()
    l0 = m.launch_count()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters, toks, comp, _ = run(reqs, False, 0)
    e1.record(stream)
    e1.synchronize()
    clk = clocks.stop()
    barrier()
    launches = m.launch_count() - l0
    dev_ms = _max_over_ranks(dist, e0.elapsed_time(e1))
    barrier()
    t0 = time.perf_counter()
    iters2, toks2, _, io = run(reqs, True, 1 << 41)
    barrier()
    wall_s = _max_over_ranks(dist, time.perf_counter() - t0)
    total = sum(r.prompt_len + r.decode_len for r in reqs)
    assert toks == total == toks2, (toks, total, toks2)
    n_hyb = sum(1 for p_, d_ in comp if p_ and d_)
    out = {
        "metric": METRIC, "value": round(toks / (dev_ms / 1e3), 1), "unit": "tokens/s", "n_gpus": world,
        "steps": iters, "warmup": args.warmup, "ms_per_step": round(dev_ms / iters, 4), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-based generator weights/tokens, seed 0; Zipf lengths)",
        "config": {"workload": args.workload, "model_shape": model_name, "requests": n_req, "B": B, "chunk": C,
                   "pd_ratio": pd, "lengths": [lo, hi], "zipf_theta": 0.4, "parallelism": f"tp{world}",
                   "kv_block_size": bs, "step": "one scheduler iteration (one run_hybrid_batch)",
                   "l2": "inputs larger than L2 (all layer weights streamed every step)"},
        "iterations": {"total": iters, "hybrid": n_hyb, "prefill_only": sum(1 for p_, d_ in comp if p_ and not d_),
                       "decode_only": sum(1 for p_, d_ in comp if d_ and not p_),
                       "mean_tokens_per_iteration": round(toks / iters, 1)},
        "e2e": {"value": round(total / wall_s, 1), "unit": "tokens/s", "makespan_s": round(wall_s, 3),
                "h2d_bytes_per_step": round(io[0] / iters2), "d2h_bytes_per_step": round(io[1] / iters2),
                "note": "per iteration: metadata H2D + logits D2H + sync (bytes: means over the run's iterations)"},
        "gpu_launches": int(launches), "gpu_launches_per_step": round(launches / iters, 1),
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    m.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# fp64 oracle on host cores (cpu_baseline leg and the --impl reference arm)
# ---------------------------------------------------------------------------
def _oracle_sample(cfg, p, s, d, ctx):
    """The identical composition for the fp64 oracle, one full-width layer: all p chunk rows
    (positions s .. s+p-1, attending the request's own prefix + chunk) and all d decode rows
    (position ctx-1, each attending its own ctx keys).  Weights: layer 0 of the generator spec.
    Residual inputs and the K/V contexts are seeded random values of the exact shapes (the prefix
    KV values do not change the work; regenerating them by running the prefix through the layer
    would cost ~100x the timed region).  LM head: every 16th vocab row, scaled to V rows."""
    import synth
    from oracle import model as om
    lw = om.layer_weights(cfg, 0, 0)
    rng = np.random.default_rng(0)
    rows_pos = [s + i for i in range(p)] + [ctx - 1] * d
    h_in = rng.standard_normal((len(rows_pos), cfg.hidden))
    kp = rng.standard_normal((s + p, cfg.n_kv_heads, cfg.head_dim))     # the chunk request's cache
    vp = rng.standard_normal((s + p, cfg.n_kv_heads, cfg.head_dim))
    base_k = rng.standard_normal((ctx, cfg.n_kv_heads, cfg.head_dim))
    base_v = rng.standard_normal((ctx, cfg.n_kv_heads, cfg.head_dim))
    scale = 1.0 + 1e-3 * np.arange(d)[:, None, None, None]
    kd = base_k[None] * scale                                            # d distinct decode caches
    vd = base_v[None] * scale
    kc = [kp[:ps + 1] for ps in rows_pos[:p]] + [kd[j] for j in range(d)]
    vc = [vp[:ps + 1] for ps in rows_pos[:p]] + [vd[j] for j in range(d)]
    wlm = synth.as_f64(synth.lm_head_rows_bits(cfg, 0, range(0, cfg.vocab, 16)))
    gf = synth.as_f64(synth.final_gain_bits(cfg, 0))
    return lw, np.array(rows_pos), h_in, kc, vc, wlm, gf


def _oracle_time(cfg, sample, reps_budget_s, decode_rows):
    """Best-of-repeats time of one full-width layer over the sample's rows + the LM head on the
    R = decode_rows + 1 logit rows (sampled vocab rows, scaled), projected to n_layers."""
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
    rows = np.r_[len(pos) - decode_rows - 1, np.arange(len(pos) - decode_rows, len(pos))]
    a = time.perf_counter()
    om.logits_rows(cfg, gf, wlm, h[rows])
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


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, p, s, d, ctx, budget_s=10.0):
    t0 = time.perf_counter()
    sample = _oracle_sample(cfg, p, s, d, ctx)
    gen_s = time.perf_counter() - t0
    tps, layer_s, head_s = _oracle_time(cfg, sample, budget_s, d)
    single = None
    try:  # one repeat with the BLAS pool limited to one thread
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            tps1, layer1, _ = _oracle_time(cfg, sample, 0.0, d)
        single = {"value": round(tps1, 3), "layer_s": round(layer1, 3)}
    except Exception as e:  # noqa: BLE001
        single = {"error": str(e)[:120]}
    n = len(sample[1])
    return {"value": round(tps, 3), "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
            "sample": (f"one full-width {cfg.name} layer (fp64 NumPy oracle) over all {n} rows of the bench "
                       f"composition ({p} chunk rows at prefix {s}..{s + p - 1}, {d} decode rows at ctx {ctx}), "
                       f"best of repeats within {budget_s:.0f}s, projected x{cfg.n_layers} layers + LM head "
                       f"({d + 1} rows, every 16th vocab row, scaled); layer {layer_s:.3f}s, head {head_s:.3f}s; "
                       f"input generation {gen_s:.1f}s excluded"),
            "single_thread": single, "cpu_model": _cpu_model(), "host_cpu_count": os.cpu_count()}


def reference(args):
    """The base contract's reference arm for this tier: the fp64 oracle timed on the host cores, on
    the SAME config / metric / unit as our arm; one step = one full-width layer over all rows of the
    composition (+ LM head), projected to the model's layers (a bounded sample of one iteration)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    if args.workload in ZIPF_WORKLOADS:
        print(json.dumps({"impl": "reference", "unavailable": "the request-workload arm has no bounded "
                          "oracle sample (fixed compositions only)"}), flush=True)
        return
    model_name, p, s, d, ctx = WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    sample = _oracle_sample(cfg, p, s, d, ctx)
    for _ in range(args.warmup):
        _oracle_time(cfg, sample, 0.0, d)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tps, layer_s, head_s = _oracle_time(cfg, sample, 0.0, d)
        vals.append(tps)
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    n = len(sample[1])
    out = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall * 1e3 / max(args.steps, 1), 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based generator weights/tokens, seed 0)",
        "config": {"workload": args.workload, "model_shape": model_name, "p": p, "s": s, "d": d, "ctx": ctx,
                   "chunk": 256, "T": p + d, "parallelism": "tp1", "kv_block_size": 64,
                   "l2": "inputs larger than L2 (all layer weights streamed every step)"},
        "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
                         "sample": f"per step: one full-width {cfg.name} layer over all {n} rows of the composition "
                                   f"+ LM head ({d + 1} rows, sampled vocab rows scaled), projected to "
                                   f"{cfg.n_layers} layers (fp64 NumPy oracle)", "cpu_model": _cpu_model()},
        "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS) + sorted(ZIPF_WORKLOADS))
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

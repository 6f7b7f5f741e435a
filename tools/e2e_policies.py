"""End-to-end scheduling-policy comparison on one B200 (§5.2, P:L51-66 and P:L85-104;
SURVEY §8(d) config 3 / §8(f) NEXT-3).

Every request has the same (P, D) = split(length, P:D) (the paper's uniform-request setup,
P:L503); B = the largest batch whose (P+D)-token KV reservations fit (sarathi_max_batch);
N = n_factor * B requests arrive at t = 0.  The same C-ABI model and host scheduler run
  * sarathi        : decode-maximal batches, chunk C = 256, <= B-1 piggybacked decodes
  * request_level  : the baseline — each prompt as its own prefill-only batch, then decode-only
                     batches of the running cohort
  * orca_best      : iteration-level batching with whole prompts (Orca best case)
  * sarathi_b200   : sarathi with the chunk chosen per iteration by sarathi_chunk_advice (B200
                     tile-quantization rule)
End-to-end throughput = sum_r (P_r + D_r) / makespan (wall clock around the whole run, device
synchronised at the end; every batch also computes the LM head for its returned rows).

Roofline counterfactual (round 2): every iteration's composition (chunk p at prefix s, decode
contexts) is also priced at the machine's roofline with the measured peaks (MEASURED_PEAKS.json:
sustained bf16 tensor FLOP/s, HBM copy GB/s): per layer max(2 T W / F, 2 W / B) for the linears +
max(FLOPs / F, KV bytes / B) for the chunk's attention + decode KV bytes / B, plus the LM head.
roofline tokens/s = sum_r (P_r + D_r) / sum of the iterations' roofline times.  The ratio of
policies at roofline says what the machine balance alone predicts; the measured ratio what this
implementation achieves.

    python tools/e2e_policies.py [--model llama-33b] [--lengths 1024] [--pd 10] [--n-factor 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def roofline_iter_s(cfg, p, s, dec_ctx, peaks):
    """Roofline time of one hybrid batch on one GPU (seconds)."""
    F = peaks["bf16_tflops_sustained"] * 1e12
    Bw = peaks["hbm_gbs"] * 1e9
    W = cfg.params_per_layer()
    T = p + len(dec_ctx)
    hd, nq, nkv = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    t_lin = max(2.0 * T * W / F, 2.0 * W / Bw)
    t_pre = 0.0
    if p:
        fl = 4.0 * hd * nq * (p * s + p * (p + 1) / 2)
        by = (s + p) * 2 * nkv * hd * 2
        t_pre = max(fl / F, by / Bw)
    t_dec = sum(dec_ctx) * 2 * nkv * hd * 2 / Bw
    R = len(dec_ctx) + (1 if p else 0)
    t_head = max(2.0 * R * cfg.vocab * cfg.hidden / F, 2.0 * cfg.vocab * cfg.hidden / Bw)
    return cfg.n_layers * (t_lin + t_pre + t_dec) + t_head


def run_policy(S, synth, torch, m, cfg, policy, P, D, N, B, C, num_blocks, bs, stream, peaks=None):
    policy, tile = policy if isinstance(policy, tuple) else (policy, 0)
    sched = S.Scheduler(B, C, num_blocks, bs, policy=policy, tile_adjust=tile)
    for r in range(N):
        sched.submit(r, P, D, 0)
    logits = torch.empty((B + 1, cfg.vocab), dtype=torch.float32, device="cuda")
    V = cfg.vocab
    tok = lambda r, a, n=1: synth.tokens(11, r, a, n, V)
    iters = 0
    roof = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while not sched.done():
        plan, admitted = sched.next()
        for rid in admitted:
            m.request_alloc(rid, P + D)
        if plan is None:
            sched.idle_step()
            continue
        pre, decs = plan
        prefill = (pre[0], pre[1], tok(pre[0], pre[1], pre[2])) if pre is not None else None
        decodes = [(rid, int(tok(rid, pos)[0]), pos) for rid, pos in decs]
        m.run_hybrid_batch(prefill, decodes, logits_ptr=logits.data_ptr())
        iters += 1
        if peaks:
            roof += roofline_iter_s(cfg, pre[2] if pre else 0, pre[1] if pre else 0, [pos + 1 for _, pos in decs], peaks)
        for rid in sched.complete():
            m.request_free(rid)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, iters, roof


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-33b")
    ap.add_argument("--lengths", type=int, nargs="*", default=[1024])
    ap.add_argument("--pd", type=float, nargs="*", default=[10.0])
    ap.add_argument("--n-factor", type=float, default=2.0)
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--policies", nargs="*", default=["sarathi", "request_level", "orca_best"])
    ap.add_argument("--pd-optimal", action="store_true",
                    help="per length, P:D = C / (B - 1) (the paper's balanced ratio, P:L62 / P:L100) instead of --pd")
    args = ap.parse_args()
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    cfg = synth.CONFIGS[args.model]
    stream = torch.cuda.Stream()
    bs = 64
    pol = {"sarathi": S.POLICY_SARATHI, "request_level": S.POLICY_REQUEST_LEVEL, "orca_best": S.POLICY_ORCA_BEST,
           "sarathi_b200": (S.POLICY_SARATHI, 2),  # chunk per iteration by the B200 advisor
           # Orca worst case: all requests begin and end together, no prefill/decode overlap,
           # "similar to our earlier baseline" -- the request-level cohort schedule
           "orca_worst": S.POLICY_REQUEST_LEVEL}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    rows = []
    for L in args.lengths:
        m = S.Model(S.config_from(cfg, max_tokens_per_batch=max(L, args.chunk) + 512), seed=0, stream=stream.cuda_stream)
        B = m.max_batch(L, reserve_bytes=8 << 30)
        per_req_blocks = -(-L // bs)
        num_blocks = B * per_req_blocks + 8
        m.alloc_kv(num_blocks, bs)
        N = max(B, int(args.n_factor * B))
        for r in ([args.chunk / max(1, B - 1)] if args.pd_optimal else args.pd):
            P, D = synth.split_pd(L, r)
            res = {}
            for name in args.policies:
                wall, iters, roof = run_policy(S, synth, torch, m, cfg, pol[name], P, D, N, B, args.chunk, num_blocks,
                                               bs, stream, peaks)
                res[name] = {"makespan_s": round(wall, 3), "iterations": iters,
                             "tokens_per_s": round(N * (P + D) / wall, 1),
                             "roofline_tokens_per_s": round(N * (P + D) / roof, 1),
                             "frac_of_roofline": round(roof / wall, 3)}
            row = {"model": args.model, "length": L, "pd_ratio": r, "P": P, "D": D, "B": B, "N": N,
                   "chunk": args.chunk, **res}
            if "request_level" in res:
                for name in res:
                    if name != "request_level":
                        row[f"speedup_{name}_vs_request_level"] = round(res[name]["tokens_per_s"] /
                                                                         res["request_level"]["tokens_per_s"], 3)
                        row[f"roofline_speedup_{name}_vs_request_level"] = round(
                            res[name]["roofline_tokens_per_s"] / res["request_level"]["roofline_tokens_per_s"], 3)
            rows.append(row)
            print(json.dumps(row), flush=True)
        m.close()
        del m


if __name__ == "__main__":
    main()

"""Chunk-size / tile-quantization sweep on B200 (§4.4 "identifying the ideal chunk size"
P:L432-463, §5.1.4 op breakdown P:L70-80, §5.4 chunked-prefill overhead P:L540-554;
SURVEY §8(f) NEXT-2).

LLaMA-13B, one P-token prompt (default 2048) prefilled in chunks while d decodes (context 1024)
ride along in every iteration, for chunk sizes C in {64, 128, 192, 256, 320, 384, 512} and three
chunk rules (the scheduler's tile_adjust modes):
  literal : p = C
  paper   : p = C - d            (chunk + decodes = C, the paper's tile-adjusted chunk)
  b200    : p = chunk_advice(C, d, remaining)   (the same rule on this GEMM's token quanta)
Per (C, rule): the whole prompt's iterations are timed (CUDA events, median of --reps per
iteration), giving prompt time, hybrid tokens/s = (P + iterations * d) / time, and the per-op
breakdown (preproj = QKV GEMM, attention = prefill + decode attention, postproj = O GEMM,
ffn = gate||up + down GEMMs, others) from a separate profiled pass (per-op events break the PDL
chains, so the breakdown sums to slightly more than the timed total).  The unchunked reference is
the full prompt as ONE prefill-only batch (T = P) with the decodes as their own decode-only batch.

    python tools/chunk_sweep.py [--prompt 2048] [--ds 16 64] [--chunks 64 128 ...] [--reps 3]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GROUPS = {"preproj": ["gemm_qkv"], "attention": ["prefill_attn", "decode_attn"], "postproj": ["gemm_o"],
          "ffn": ["gemm_gate_up", "gemm_down"], "others": ["embed", "rmsnorm", "lm_head", "allreduce", "other"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompt", type=int, default=2048)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--ds", type=int, nargs="*", default=[16, 64])
    ap.add_argument("--chunks", type=int, nargs="*", default=[64, 128, 192, 256, 320, 384, 512])
    ap.add_argument("--rules", nargs="*", default=["literal", "paper", "b200"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    cfg = synth.LLAMA_13B
    P, ctx = args.prompt, args.ctx
    dmax = max(args.ds)
    stream = torch.cuda.Stream()
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=P + dmax), seed=0, stream=stream.cuda_stream)
    bs = 64
    m.alloc_kv((dmax + 1) * -(-max(P, ctx) // bs) + 8, bs)
    tok = lambda r, a, n: synth.tokens(7, r, a, n, cfg.vocab)
    m.request_alloc(0, P)
    for r in range(1, dmax + 1):
        m.request_alloc(r, ctx)
        for a in range(0, ctx - 1, 1024):
            m.run_hybrid_batch((r, a, tok(r, a, min(1024, ctx - 1 - a))), [], flags=S.NO_LOGITS)
    logits = torch.empty((dmax + 1, cfg.vocab), dtype=torch.float32, device="cuda")

    def run(pre, decs, reps):
        ts = []
        for _ in range(reps):
            if pre is not None:
                m.truncate(0, pre[1])
            for r, _, pos in decs:
                m.truncate(r, pos)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            m.run_hybrid_batch(pre, decs, logits_ptr=logits.data_ptr())
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def plan(C, d, rule):
        out, s = [], 0
        while s < P:
            rem = P - s
            if rule == "literal":
                p = min(C, rem)
            elif rule == "paper":
                p = min(max(1, C - d), rem)
            else:
                p = S.chunk_advice(C, d, rem)
            out.append((s, p))
            s += p
        return out

    rows = []
    for d in args.ds:
        decs = [(r, int(tok(r, ctx - 1, 1)[0]), ctx - 1) for r in range(1, d + 1)]
        # unchunked reference: the whole prompt as one prefill-only batch + one decode-only batch
        for _ in range(2):
            run((0, 0, tok(0, 0, P)), [], 1)
        t_full = run((0, 0, tok(0, 0, P)), [], args.reps)
        t_dec = run(None, decs, args.reps)
        ref = {"d": d, "rule": "unchunked", "chunk": P, "iterations": 2, "prompt_ms": round(t_full, 3),
               "decode_only_ms": round(t_dec, 3), "total_ms": round(t_full + t_dec, 3),
               "tokens_per_s": round((P + d) / ((t_full + t_dec) / 1e3), 1)}
        rows.append(ref)
        print(json.dumps(ref), flush=True)
        for C in args.chunks:
            for rule in args.rules:
                pl = plan(C, d, rule)
                run((0, pl[0][0], tok(0, pl[0][0], pl[0][1])), decs, 1)  # warm the GEMM plans / maps
                times = [run((0, s, tok(0, s, p)), decs, args.reps) for s, p in pl]
                m.set_profiling(True)
                m.op_times(reset=True)
                for s, p in pl:
                    run((0, s, tok(0, s, p)), decs, 1)
                ops = m.op_times(reset=True)
                m.set_profiling(False)
                total = sum(times)
                br = {g: round(sum(ops[k][0] for k in ks), 3) for g, ks in GROUPS.items()}
                chunks = sorted({p for _, p in pl})
                row = {"d": d, "rule": rule, "chunk": C, "chunk_sizes": chunks[:4] + (["..."] if len(chunks) > 4 else []),
                       "T_first": pl[0][1] + d, "token_capacity": S.token_capacity(pl[0][1] + d)[0],
                       "iterations": len(pl), "prompt_ms": round(total, 3),
                       "tokens_per_s": round((P + len(pl) * d) / (total / 1e3), 1),
                       "ms_per_iteration": round(total / len(pl), 3),
                       "prefill_overhead_vs_unchunked": round(total / t_full, 3),
                       "breakdown_ms": br}
                rows.append(row)
                print(json.dumps(row), flush=True)
    # summary table
    print("\n| d | rule | C | iters | T (first) | capacity | prompt ms | tok/s | x unchunked prompt | preproj | attn | postproj | ffn | others |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        if r["rule"] == "unchunked":
            print(f"| {r['d']} | unchunked | {r['chunk']} | 1+1 | {r['chunk']} | | {r['prompt_ms']} (+{r['decode_only_ms']} decode) "
                  f"| {r['tokens_per_s']} | 1.0 | | | | | |")
            continue
        b = r["breakdown_ms"]
        print(f"| {r['d']} | {r['rule']} | {r['chunk']} | {r['iterations']} | {r['T_first']} | {r['token_capacity']} | "
              f"{r['prompt_ms']} | {r['tokens_per_s']} | {r['prefill_overhead_vs_unchunked']} | {b['preproj']} | "
              f"{b['attention']} | {b['postproj']} | {b['ffn']} | {b['others']} |")
    m.close()


if __name__ == "__main__":
    main()

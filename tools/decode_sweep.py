"""Decode-maximal batching microbenchmark on B200 (§5.1, Fig. "decode speedup", P:L32-35;
SURVEY §8(d) config 2; BASELINE.json metric "marginal decode ms/token").

For LLaMA-13B at prompt length P in {1024, 2048, 3072}: one prefill chunk of 256 tokens (the last
chunk of a P-token prompt, cached prefix P-256) piggybacked with d decodes at context P, for d up to
B-1 (B from sarathi_max_batch at reservation P + 128, reading O-18):
    marginal decode ms/token = (t(chunk + d decodes) - t(chunk alone)) / d
    decode-only ms/token     =  t(d decodes alone) / d                            (baseline batch)
    decode speedup           =  decode-only / marginal
Every time is the median of CUDA-event-timed hybrid batches (requests rolled back between steps),
inputs resident in HBM.  Prints one JSON line per (P, d) and a summary table.

    python tools/decode_sweep.py [--prompts 1024 2048 3072] [--ds 1 2 4 8 16 32 64 128 -1] [--steps 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, nargs="*", default=[1024, 2048, 3072])
    ap.add_argument("--ds", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32, 64, 128, -1])
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    cfg = synth.LLAMA_13B
    stream = torch.cuda.Stream()
    rows = []
    for P in args.prompts:
        C = args.chunk
        m = S.Model(S.config_from(cfg, max_tokens_per_batch=512), seed=0, stream=stream.cuda_stream)
        bs = 64
        B = m.max_batch(P + 128, reserve_bytes=8 << 30)
        dmax = max(1, B - 1)
        ds = sorted({dmax if d < 0 else min(d, dmax) for d in args.ds})
        nd = max(ds)
        m.alloc_kv((nd + 1) * -(-(P + 128) // bs) + 8, bs)
        tok = lambda r, a, n: synth.tokens(7, r, a, n, cfg.vocab)
        # request 0: the prefill request at cached prefix P - C; 1..nd: decoders at context P
        s = P - C
        m.request_alloc(0, P + 128)
        for a in range(0, s, 512):
            m.run_hybrid_batch((0, a, tok(0, a, min(512, s - a))), [], flags=S.NO_LOGITS)
        for r in range(1, nd + 1):
            m.request_alloc(r, P + 128)
            for a in range(0, P - 1, 512):
                m.run_hybrid_batch((r, a, tok(r, a, min(512, P - 1 - a))), [], flags=S.NO_LOGITS)
        pre = (0, s, tok(0, s, C))
        logits = torch.empty((nd + 1, cfg.vocab), dtype=torch.float32, device="cuda")

        def timed(prefill, decs):
            def step():
                if prefill is not None:
                    m.truncate(0, s)
                for r, _, pos in decs:
                    m.truncate(r, pos)
                m.run_hybrid_batch(prefill, decs, logits_ptr=logits.data_ptr())
            for _ in range(3):
                step()
            ts = []
            for _ in range(args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            return float(np.median(ts))

        t_chunk = timed(pre, [])
        for d in ds:
            decs = [(r, int(tok(r, P - 1, 1)[0]), P - 1) for r in range(1, d + 1)]
            t_hyb = timed(pre, decs)
            t_dec = timed(None, decs)
            # tile-adjusted chunk (§4.4, reading O-15): p = C - d so T = C
            t_tile = timed((0, s, tok(0, s, C - d)), decs) if 0 < d < C else None
            marg = (t_hyb - t_chunk) / d
            base = t_dec / d
            row = {"model": "llama-13b", "P": P, "chunk": C, "d": d, "B": B, "t_hybrid_ms": round(t_hyb, 3),
                   "t_chunk_only_ms": round(t_chunk, 3), "t_decode_only_ms": round(t_dec, 3),
                   "marginal_decode_ms_per_token": round(marg, 4), "decode_only_ms_per_token": round(base, 4),
                   "decode_speedup": round(base / marg, 2) if marg > 0 else None,
                   "hybrid_tokens_per_s": round((C + d) / t_hyb * 1e3, 1),
                   "tile_adjusted": ({"p": C - d, "t_ms": round(t_tile, 3),
                                      "hybrid_tokens_per_s": round(C / t_tile * 1e3, 1)} if t_tile else None)}
            rows.append(row)
            print(json.dumps(row), flush=True)
        m.close()
        del m
    print("\n| P | d | B | hybrid ms | chunk-only ms | decode-only ms | marginal ms/tok | decode-only ms/tok | speedup | hybrid tok/s | tile-adj. p=C-d tok/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        ta = r["tile_adjusted"]["hybrid_tokens_per_s"] if r["tile_adjusted"] else "-"
        print(f"| {r['P']} | {r['d']} | {r['B']} | {r['t_hybrid_ms']} | {r['t_chunk_only_ms']} | {r['t_decode_only_ms']} | "
              f"{r['marginal_decode_ms_per_token']} | {r['decode_only_ms_per_token']} | {r['decode_speedup']} | "
              f"{r['hybrid_tokens_per_s']} | {ta} |")
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Pipeline bubbles on B200 with measured stage times (§5.3, L311-327 §3.2; SURVEY
§8(f) NEXT-4).  The paper simulated GPT-3 on 64 A100s (TP-8 x PP-8) from profiled op times; here the
per-layer time of every micro-batch composition is MEASURED on one B200 (the GPT-3 TP-8 rank shard:
12 heads, H = 12288, 2-matrix GELU FFN of 6144 rows), fitted as

    t_layer(p, s, ctx) = c0 + c1 * T + c2 * p * (s + p / 2) + c3 * sum(ctx)        (T = p + d)

(least squares over a grid of prefill / decode / hybrid compositions; the fit error is printed),
and the 8-stage pipeline is replayed with paper_2308_16369_b200.pipeline.pipeline_timeline for the
micro-batches the C++ scheduler forms (8 in-flight groups of <= B requests, Zipf(0.4) lengths
1K-4K, P:D = 10, chunk 256) under Orca-best (whole prompts) and SARATHI (chunk + piggybacked
decodes).  Reports the per-request bubble time (median, p90) and the makespan of each policy.
Not measured: the TP all-reduces and the stage-to-stage activation sends (identical under both
policies for the same tokens).

    python tools/pp_bubbles.py [--requests 256] [--stages 8] [--B 27] [--chunk 256]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure_costs(S, synth, torch, cfg, steps=5):
    """Per-layer ms of a grid of compositions on the rank-shard model (2 layers)."""
    stream = torch.cuda.Stream()
    maxT = 2048 + 32
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=maxT, max_seq_len=4096), seed=0, stream=stream.cuda_stream)
    bs = 64
    nd = 27
    prefixes = (0, 1024, 2048)
    ctxs = (1024, 2048, 3072, 4096)
    m.alloc_kv((nd * len(ctxs) + len(prefixes)) * (4096 // bs) + 8, bs)
    tok = lambda r, a, n: synth.tokens(7, r, a, n, cfg.vocab)
    # nd decode requests per context length (cached ctx - 1 tokens; a timed step truncates back)
    dec_req = {}
    for i, cx in enumerate(ctxs):
        dec_req[cx] = list(range(1000 * (i + 1), 1000 * (i + 1) + nd))
        for r in dec_req[cx]:
            m.request_alloc(r, 4096)
            for a in range(0, cx - 1, 2048):
                m.run_hybrid_batch((r, a, tok(r, a, min(2048, cx - 1 - a))), [], flags=S.NO_LOGITS)
    # one chunk request per prefix length s (its cache stays >= s: every timed step truncates back to s)
    pre_req = {}
    for i, s0 in enumerate(prefixes):
        rid = 100 + i
        pre_req[s0] = rid
        m.request_alloc(rid, 4096)
        for a in range(0, s0, 2048):
            m.run_hybrid_batch((rid, a, tok(rid, a, min(2048, s0 - a))), [], flags=S.NO_LOGITS)
    logits = torch.empty((maxT, cfg.vocab), dtype=torch.float32, device="cuda")
    rows = []

    def timed(p, s, d, ctx):
        rid = pre_req[s]
        pre = (rid, s, tok(rid, s, p)) if p else None
        decs = [(r, int(tok(r, ctx - 1, 1)[0]), ctx - 1) for r in dec_req[ctx][:d]] if d else []

        def step():
            if p:
                m.truncate(rid, s)
            for r, _, pos in decs:
                m.truncate(r, pos)
            m.run_hybrid_batch(pre, decs, logits_ptr=logits.data_ptr())
        step()
        ts = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts) / cfg.n_layers

    for p in (64, 128, 256, 512, 1024, 2048):
        for s in (0, 1024):
            rows.append((p, s, 0, 0, timed(p, s, 0, 1024)))
    for d in (1, 4, 11, 27):
        for ctx in (1024, 2048, 4096):
            rows.append((0, 0, d, ctx, timed(0, 0, d, ctx)))
    for s in (0, 1024, 2048):
        for d in (1, 10, 26):
            for ctx in (1024, 3072):
                rows.append((256, s, d, ctx, timed(256, s, d, ctx)))
    m.close()
    return rows


def fit(rows):
    import numpy as np
    A = np.array([[1.0, p + d, p * (s + p / 2.0), d * ctx] for p, s, d, ctx, _ in rows])
    y = np.array([t for *_, t in rows])
    c, *_ = np.linalg.lstsq(A, y, rcond=None)
    pred = A @ c
    return c, float(np.max(np.abs(pred - y) / y))


def schedule(S, synth, reqs, groups, B, C, policy, tile, num_blocks, bs):
    """Micro-batches of `groups` in-flight request groups (round-robin assignment), interleaved
    slot by slot: micro-batch m is iteration m // groups of group m % groups."""
    scheds = [S.Scheduler(B, C, num_blocks, bs, policy=policy, tile_adjust=tile) for _ in range(groups)]
    for i, r in enumerate(reqs):
        scheds[i % groups].submit(r.req_id, r.prompt_len, r.decode_len, 0)
    mbs = []  # (composition (p, s, [ctx]), [request ids])
    live = [True] * groups
    while any(live):
        for g, sc in enumerate(scheds):
            if not live[g]:
                mbs.append(((0, 0, []), []))  # an exhausted slot: empty micro-batch (costs nothing)
                continue
            if sc.done():
                live[g] = False
                mbs.append(((0, 0, []), []))
                continue
            plan, _ = sc.next()
            while plan is None:
                sc.idle_step()
                plan, _ = sc.next()
            pre, decs = plan
            ids = ([pre[0]] if pre else []) + [r for r, _ in decs]
            mbs.append(((pre[2] if pre else 0, pre[1] if pre else 0, [pos + 1 for _, pos in decs]), ids))
            sc.complete()
    while mbs and not mbs[-1][1]:
        mbs.pop()
    return mbs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=256)
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--B", type=int, default=27)
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--layers", type=int, default=96)
    args = ap.parse_args()
    import numpy as np
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S
    from paper_2308_16369_b200.pipeline import pipeline_timeline, request_bubbles

    torch.cuda.set_device(0)
    cfg = synth.ModelConfig("gpt3-tp8-rank", 2, 12288, 12, 12, 128, 6144, 6288, ffn_kind=synth.FFN_GELU,
                            max_seq_len=4096)
    rows = measure_costs(S, synth, torch, cfg)
    c, err = fit(rows)
    print(json.dumps({"cost_model_ms_per_layer": {"c0": c[0], "c1_per_token": c[1], "c2_per_prefill_attn_pair": c[2],
                                                  "c3_per_decode_ctx_token": c[3]}, "max_rel_fit_error": round(err, 4),
                      "points": len(rows)}), flush=True)
    per_stage_layers = args.layers / args.stages
    reqs = synth.zipf_workload(7, args.requests, 10.0)
    out = {}
    for name, pol, tile in (("orca_best", S.POLICY_ORCA_BEST, 0), ("sarathi", S.POLICY_SARATHI, 0),
                            ("sarathi_b200", S.POLICY_SARATHI, 2)):
        mbs = schedule(S, synth, reqs, args.stages, args.B, args.chunk, pol, tile, args.B * 64 + 64, 64)
        t = []
        for (p, s, ctx), ids in mbs:
            if not ids:
                t.append(0.0)
                continue
            tl = c[0] + c[1] * (p + len(ctx)) + c[2] * p * (s + p / 2.0) + c[3] * sum(ctx)
            t.append(per_stage_layers * tl)
        _, fin, bub = pipeline_timeline(t, args.stages)
        rb = request_bubbles([ids for _, ids in mbs], bub)
        vals = sorted(rb.values())
        tokens = sum(r.prompt_len + r.decode_len for r in reqs)
        out[name] = {"micro_batches": sum(1 for _, ids in mbs if ids), "makespan_s": round(fin[-1][-1] / 1e3, 3),
                     "tokens_per_s_per_pipeline": round(tokens / (fin[-1][-1] / 1e3), 1),
                     "bubble_ms_per_request_median": round(statistics.median(vals), 2),
                     "bubble_ms_per_request_p90": round(vals[int(0.9 * (len(vals) - 1))], 2),
                     "stage_time_cv": round(float(np.std([x for x in t if x > 0]) / np.mean([x for x in t if x > 0])), 3)}
        print(json.dumps({name: out[name]}), flush=True)
    print(json.dumps({"median_bubble_reduction_sarathi_vs_orca_best":
                      round(out["orca_best"]["bubble_ms_per_request_median"] /
                            max(out["sarathi"]["bubble_ms_per_request_median"], 1e-9), 2),
                      "paper": "6.29x lower median bubble per request (simulated 64 x A100, P:L18)",
                      "config": {"model": "GPT-3 175B shape, TP-8 rank shard, " + str(args.layers) + " layers",
                                 "stages": args.stages, "B": args.B, "chunk": args.chunk, "requests": args.requests,
                                 "workload": "Zipf(0.4) 1K-4K, P:D = 10"}}), flush=True)


if __name__ == "__main__":
    main()

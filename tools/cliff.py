"""Per-op device spans of hybrid batches around the 256-token GEMM boundary (§4.4 tile
quantization): LLaMA-13B, the last 256-token chunk of a 1K prompt with d decodes at
context 1024, for (p, d) in --cases; prints step time (CUDA events) and every op's mean device span.

    python tools/cliff.py [--cases 256:0 256:1 255:1 256:16 240:16]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="*", default=["256:0", "256:1", "255:1", "256:16", "240:16"])
    ap.add_argument("--steps", type=int, default=8)
    args = ap.parse_args()
    import torch
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    cfg = synth.LLAMA_13B
    stream = torch.cuda.Stream()
    P, bs = 1024, 64
    nd = max(int(c.split(":")[1]) for c in args.cases)
    m = S.Model(S.config_from(cfg, max_tokens_per_batch=512), seed=0, stream=stream.cuda_stream)
    m.alloc_kv((nd + 1) * (P // bs + 2) + 8, bs)
    tok = lambda r, a, n: synth.tokens(7, r, a, n, cfg.vocab)
    m.request_alloc(0, P)
    m.run_hybrid_batch((0, 0, tok(0, 0, 512)), [], flags=S.NO_LOGITS)
    m.run_hybrid_batch((0, 512, tok(0, 512, 256)), [], flags=S.NO_LOGITS)
    for r in range(1, nd + 1):
        m.request_alloc(r, P)
        m.run_hybrid_batch((r, 0, tok(r, 0, 512)), [], flags=S.NO_LOGITS)
        m.run_hybrid_batch((r, 512, tok(r, 512, 511)), [], flags=S.NO_LOGITS)
    logits = torch.empty((nd + 1, cfg.vocab), dtype=torch.float32, device="cuda")
    for case in args.cases:
        p, d = (int(x) for x in case.split(":"))
        pre = (0, 768, tok(0, 768, p)) if p else None
        decs = [(r, int(tok(r, P - 1, 1)[0]), P - 1) for r in range(1, d + 1)]

        def step():
            m.truncate(0, 768)
            for r, _, pos in decs:
                m.truncate(r, pos)
            m.run_hybrid_batch(pre, decs, logits_ptr=logits.data_ptr())
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
        m.set_profiling(True)
        m.op_times(reset=True)
        m.op_kernel_times(reset=True)
        for _ in range(args.steps):
            step()
        kops = m.op_kernel_times(reset=True)
        ops = m.op_times(reset=True)
        m.set_profiling(False)
        print(json.dumps({"p": p, "d": d, "T": p + d, "ms": round(statistics.median(ts), 4),
                          "span_us": {k: round(v[0] / v[1] * 1e3, 2) for k, v in kops.items() if v[1]},
                          "event_us": {k: round(v[0] / v[1] * 1e3, 2) for k, v in ops.items() if v[1]}}), flush=True)
    m.close()


if __name__ == "__main__":
    main()

"""Per-rank compute of a tensor-parallel hybrid batch on ONE B200 (no all-reduce): the per-GPU
GEMM / attention shapes of a TP-t rank (SURVEY §8(a) [70B-8]; §8(e)), as a single-GPU model whose
heads / FFN / vocab are the rank's shard.  Reports the step time and tokens/s of the rank's
compute; the two all-reduces per layer (T x H x 2 B each) are NOT included (1-GPU boxes).

    python tools/shard_step.py [--which llama70b-tp8 llama13b-tp8 gpt3-tp8] [--layers 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", nargs="*", default=["llama70b-tp8", "llama13b-tp8", "gpt3-tp8"])
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    L = args.layers
    shards = {  # rank shapes (heads/t, H2/t, V/t) and the SURVEY compositions
        "llama70b-tp8": (synth.ModelConfig("llama2-70b-tp8-rank", L, 8192, 8, 1, 128, 3584, 4000, max_seq_len=2048),
                         256, 1024, 26, 2048, 80),
        "llama13b-tp8": (synth.ModelConfig("llama-13b-tp8-rank", L, 5120, 5, 5, 128, 1728, 4000, max_seq_len=1024),
                         256, 768, 64, 1024, 40),
        "gpt3-tp8": (synth.ModelConfig("gpt3-tp8-rank", L, 12288, 12, 12, 128, 6144, 6288, ffn_kind=synth.FFN_GELU,
                                       max_seq_len=2048), 256, 1024, 26, 2048, 96),
    }
    for name in args.which:
        cfg, p, s, d, ctx, L_full = shards[name]
        stream = torch.cuda.Stream()
        m, prefill, decodes = bench.setup_model(S, synth, cfg, p, s, d, ctx, 0, 1, 0, None, stream.cuda_stream)
        logits = torch.empty((d + 1, cfg.vocab), dtype=torch.float32, device="cuda")

        def step():
            m.truncate(prefill[0], prefill[1])
            for r, _, pos in decodes:
                m.truncate(r, pos)
            m.run_hybrid_batch(prefill, decodes, logits_ptr=logits.data_ptr())
        for _ in range(3):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        m.set_profiling(True)
        m.op_times(reset=True)
        for _ in range(args.steps):
            step()
        ops = m.op_times(reset=True)
        kops = m.op_kernel_times(reset=True)
        m.set_profiling(False)
        per_layer = ms / L
        row = {"shard": name, "layers_run": L, "p": p, "s": s, "d": d, "ctx": ctx, "T": p + d,
               "ms_per_layer": round(per_layer, 4), "projected_ms_per_step_compute_only": round(per_layer * L_full, 3),
               "projected_tokens_per_s_compute_only": round((p + d) / (per_layer * L_full) * 1e3, 1),
               "op_us_per_layer": {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in ops.items() if v[1]},
               "kernel_span_us": {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in kops.items() if v[1]},
               "note": "one TP rank's compute on one B200; all-reduces not included"}
        print(json.dumps(row), flush=True)
        m.close()
        del m


if __name__ == "__main__":
    main()

"""Runs the bench composition and brackets N steps with cudaProfilerStart/Stop so that
`ncu --profile-from-start off ...` captures exactly those steps (setup excluded).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file out.csv \
        python tools/profile_step.py --steps 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--workload", default="llama13b-p256-s768-d64-ctx1024")
    ap.add_argument("--kind", default="hybrid", choices=["hybrid", "prefill", "decode"])
    ap.add_argument("--spans", type=int, default=0,
                    help="print the device-span timeline of the first N kernels of one profiled step "
                         "(SARATHI_SPANS_ONLY: no per-op events, the PDL chain is intact)")
    args = ap.parse_args()
    if args.spans:  # read once by the library (static), so before the first launch
        os.environ["SARATHI_SPANS_ONLY"] = "1"
        os.environ["SARATHI_SPAN_DUMP"] = str(args.spans)
    import torch
    import bench
    import synth
    from paper_2308_16369_b200 import sarathi as S

    torch.cuda.set_device(0)
    model_name, p, s, d, ctx = bench.WORKLOADS[args.workload]
    cfg = synth.CONFIGS[model_name]
    stream = torch.cuda.Stream()
    m, prefill, decodes = bench.setup_model(S, synth, cfg, p, s, d, ctx, 0, 1, 0, None, stream.cuda_stream)
    if args.kind == "prefill":
        decodes = []
    if args.kind == "decode":
        prefill = None
    logits = torch.empty((d + 1, cfg.vocab), dtype=torch.float32, device="cuda")

    def step():
        if prefill is not None:
            m.truncate(prefill[0], prefill[1])
        for r, _, pos in decodes:
            m.truncate(r, pos)
        m.run_hybrid_batch(prefill, decodes, logits_ptr=logits.data_ptr())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.spans:
        m.set_profiling(True)
        step()
        torch.cuda.synchronize()
        m.op_times(reset=True)
        ks = m.op_kernel_times(reset=True)
        print("kernel spans (ms per step):", {k: round(v[0], 4) if isinstance(v, tuple) else v for k, v in ks.items()})
        m.set_profiling(False)
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    m.close()
    print("profiled", args.steps, "step(s) of", args.workload, args.kind)


if __name__ == "__main__":
    main()

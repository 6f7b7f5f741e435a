"""Times sarathi_op_gemm (the tcgen05 GEMM through the C ABI) on the LLaMA-13B layer shapes.

    python tools/gemm_bench.py [--n 320] [--iters 20]

Prints per shape/mode: us, TFLOP/s (algorithmic 2*M*N*K), weight GB/s, fraction of the measured bf16 peak.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[64, 160, 256, 320, 512])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--modes", type=int, nargs="*", default=[0, 1])
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()
    import torch
    from paper_2308_16369_b200 import sarathi as S
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824),
              "lm_head": (32000, 5120)}
    st = torch.cuda.current_stream()
    for name, (M, K) in shapes.items():
        W0 = (torch.randn(M, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        # two packed copies, alternated back to back: > L2, so every launch streams its weights from HBM
        Ws = [torch.empty(((M + 127) // 128 * 128) * K, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        for W in Ws:
            S.op_pack_weight(W0.data_ptr(), W.data_ptr(), M, K, st.cuda_stream)
        for N in args.n:
            X = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            for mode in args.modes:
                if mode == 3:
                    out = torch.zeros(N, M // 2, device="cuda", dtype=torch.bfloat16)
                elif mode in (1, 2):
                    out = torch.zeros(N, M, device="cuda", dtype=torch.float32)
                else:
                    out = torch.zeros(N, M, device="cuda", dtype=torch.bfloat16)
                flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
                run = lambda i: S.op_gemm(Ws[i & 1].data_ptr(), X.data_ptr(), out.data_ptr(), M, N, K,
                                          mode | S.GEMM_W_PACKED, args.ctas, st.cuda_stream)
                for i in range(3):
                    run(i)
                ts = []
                reps = 8  # back-to-back launches per sample: the GPU queue stays ahead of host launch overhead
                for _ in range(args.iters):
                    flush.zero_()
                    torch.cuda._sleep(2000000)  # ~1 ms: the host enqueues every launch before the first runs
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for i in range(reps):
                        run(i)
                    e1.record(st)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) / reps)
                ts.sort()
                ms = ts[len(ts) // 2]
                fl = 2.0 * M * N * K
                print(f"{name:8s} M={M:5d} N={N:4d} K={K:5d} mode={mode}  {ms*1e3:8.1f} us  "
                      f"{fl/ms/1e9:7.1f} TFLOP/s  {2*M*K/ms/1e6:7.1f} GB/s(w)  frac={fl/ms/1e9/peaks['bf16_tflops']:.3f}",
                      flush=True)


if __name__ == "__main__":
    main()

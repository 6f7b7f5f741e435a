"""One sarathi_op_gemm launch bracketed by cudaProfilerStart/Stop (for ncu --profile-from-start off).

    python tools/gemm_one.py M N K [mode] [pairs]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2308_16369_b200 import sarathi as S
    M, N, K = (int(x) for x in sys.argv[1:4])
    mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    pairs = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    W0 = (torch.randn(M, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    W = torch.empty(((M + 127) // 128 * 128) * K, device="cuda", dtype=torch.bfloat16)
    S.op_pack_weight(W0.data_ptr(), W.data_ptr(), M, K, torch.cuda.current_stream().cuda_stream)
    mode |= S.GEMM_W_PACKED
    X = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(N, M, device="cuda", dtype=torch.float32 if mode in (1, 2) else torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        S.op_gemm(W.data_ptr(), X.data_ptr(), out.data_ptr(), M, N, K, mode, pairs, st)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    S.op_gemm(W.data_ptr(), X.data_ptr(), out.data_ptr(), M, N, K, mode, pairs, st)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()

"""GPU parity of the tcgen05 GEMM (through sarathi_op_gemm, the C ABI).

Exactness first: small-integer operands are exact in bf16 and every partial sum is an integer
< 2^24, so an fp32-accumulating GEMM must reproduce the integer product EXACTLY whatever the
UMMA descriptor / swizzle / split-K path — a mis-encoded descriptor cannot hide.  Then random
bf16 operands at the LLaMA-13B shapes against an fp64 matmul of the same bf16 values."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2308_16369_b200 import sarathi
    return sarathi


def _int_operands(M, N, K, seed):
    g = torch.Generator().manual_seed(seed)
    W = torch.randint(-3, 4, (M, K), generator=g).to(torch.bfloat16)
    X = torch.randint(-3, 4, (N, K), generator=g).to(torch.bfloat16)
    return W, X


SHAPES = [
    (128, 16, 64, 0), (128, 1, 64, 0), (256, 320, 5120, 1), (256, 320, 5120, 4), (384, 7, 128, 0),
    (200, 37, 192, 0), (128, 600, 256, 0), (1280, 282, 8192, 0), (512, 257, 1024, 3), (640, 512, 640, 2),
    # 256 < N <= 512 with one segment per CTA pair: the uneven split (UMMA N = 256 + 16-multiple tail)
    (256, 257, 256, 0), (768, 300, 512, 0), (256, 497, 128, 0), (5120, 272, 1024, 0),
    # more 256-row tiles than CTA pairs with two equal UMMAs per k-step: the remainder tiles run as
    # token-half items (one UMMA's tokens per pair), incl. a ragged second half, a ragged last row
    # tile and two whole tiles per pair before the half item
    (27648, 320, 256, 0), (19000, 300, 128, 0), (40000, 288, 64, 0),
]


@pytest.mark.parametrize("M,N,K,splits", SHAPES)
def test_gemm_exact_integers_fp32_out(S, M, N, K, splits):
    W, X = _int_operands(M, N, K, M + N + K)
    ref = X.double() @ W.double().T
    Wd, Xd = W.cuda(), X.cuda()
    out = torch.full((N, M), float("nan"), device="cuda", dtype=torch.float32)
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_STORE_F32, splits,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(out.double().cpu(), ref)


@pytest.mark.parametrize("M,N,K,splits", [(256, 320, 5120, 0), (128, 33, 256, 2)])
def test_gemm_exact_bf16_out_and_residual_add(S, M, N, K, splits):
    W, X = _int_operands(M, N, K, 5)
    ref = X.double() @ W.double().T
    Wd, Xd = W.cuda(), X.cuda()
    out = torch.empty((N, M), device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_STORE_BF16, splits, st)
    base = torch.arange(N * M, dtype=torch.float32).reshape(N, M).cuda()
    acc = base.clone()
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), acc.data_ptr(), M, N, K, S.EPI_ADD_F32, splits, st)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), ref.float().to(torch.bfloat16))
    assert torch.equal(acc.double().cpu(), base.double().cpu() + ref)


def test_gemm_silu_mul_interleaved(S):
    M, N, K = 512, 40, 256   # rows [32i, 32i+16) gate of features [16i, 16i+16), [32i+16, 32i+32) their up
    g = torch.Generator().manual_seed(3)
    W = (torch.randn(M, K, generator=g) / 16).to(torch.bfloat16)
    X = torch.randn(N, K, generator=g).to(torch.bfloat16)
    acc = (X.double() @ W.double().T).reshape(N, M // 32, 2, 16)
    gate, up = acc[:, :, 0, :], acc[:, :, 1, :]
    ref = (gate / (1 + torch.exp(-gate)) * up).reshape(N, M // 2)
    out = torch.empty((N, M // 2), device="cuda", dtype=torch.bfloat16)
    Wd, Xd = W.cuda(), X.cuda()   # keep the device tensors alive until the kernel ran
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_SILU_MUL, 0,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    err = (out.double().cpu() - ref).abs().max() / ref.abs().max()
    assert err < 1e-2


@pytest.mark.parametrize("half", ["1", "0"])
def test_gemm_silu_mul_gate_up_shape(S, half):
    """LLaMA-13B gate||up at T = 320 (108 row tiles on 74 CTA pairs): the remainder as token-half
    items (default) and as the stream-K split (SARATHI_GEMM_HALF=0, in a child process: the switch is
    read once per process)."""
    import subprocess
    import sys
    code = (
        "import torch, sys; sys.path.insert(0, '.');"
        "from paper_2308_16369_b200 import sarathi as S;"
        "M, N, K = 27648, 320, 1024;"
        "g = torch.Generator().manual_seed(11);"
        "W = (torch.randn(M, K, generator=g) / 32).to(torch.bfloat16);"
        "X = torch.randn(N, K, generator=g).to(torch.bfloat16);"
        "acc = (X.double() @ W.double().T).reshape(N, M // 32, 2, 16);"
        "gate, up = acc[:, :, 0, :], acc[:, :, 1, :];"
        "ref = (gate / (1 + torch.exp(-gate)) * up).reshape(N, M // 2);"
        "out = torch.empty((N, M // 2), device='cuda', dtype=torch.bfloat16);"
        "Wd, Xd = W.cuda(), X.cuda();"
        "S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_SILU_MUL, 0, torch.cuda.current_stream().cuda_stream);"
        "torch.cuda.synchronize();"
        "err = ((out.double().cpu() - ref).abs().max() / ref.abs().max()).item();"
        "print('err', err); assert err < 1e-2, err"
    )
    import os
    env = dict(os.environ, SARATHI_GEMM_HALF=half)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_gemm_gelu(S):
    M, N, K = 256, 24, 128
    g = torch.Generator().manual_seed(4)
    W = (torch.randn(M, K, generator=g) / 8).to(torch.bfloat16)
    X = torch.randn(N, K, generator=g).to(torch.bfloat16)
    ref = torch.nn.functional.gelu(X.double() @ W.double().T, approximate="tanh")
    out = torch.empty((N, M), device="cuda", dtype=torch.bfloat16)
    Wd, Xd = W.cuda(), X.cuda()
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_GELU, 0,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (out.double().cpu() - ref).abs().max() / ref.abs().max() < 1e-2


@pytest.mark.parametrize("M,K", [(15360, 5120), (5120, 5120), (27648, 5120), (5120, 13824), (32000, 5120)])
def test_gemm_llama13b_shapes_random(S, M, K):
    N = 320
    g = torch.Generator().manual_seed(M + K)
    W = (torch.randn(M, K, generator=g) / K ** 0.5).to(torch.bfloat16)
    X = torch.randn(N, K, generator=g).to(torch.bfloat16)
    Wd, Xd = W.cuda(), X.cuda()
    out = torch.empty((N, M), device="cuda", dtype=torch.float32)
    S.op_gemm(Wd.data_ptr(), Xd.data_ptr(), out.data_ptr(), M, N, K, S.EPI_STORE_F32, 0,
              torch.cuda.current_stream().cuda_stream)
    ref = (Xd.double() @ Wd.double().T)
    torch.cuda.synchronize()
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 5e-5, err   # fp32 accumulation over K <= 13824 terms


@pytest.mark.skipif(__import__("os").environ.get("SARATHI_GEMM_VARIANT_CHILD") == "1", reason="child process")
@pytest.mark.parametrize("env", [{"SARATHI_GEMM_KBASM": "0"}, {"SARATHI_GEMM_RELAXED": "0"}])
def test_gemm_issue_variants(env):
    """The per-UMMA issue path (SARATHI_GEMM_KBASM=0) and release-semantics TMEM-slot arrives
    (SARATHI_GEMM_RELAXED=0), read once per process, rerun the exact-integer shapes in a child."""
    import os
    import subprocess
    import sys
    e = dict(os.environ, SARATHI_GEMM_VARIANT_CHILD="1", **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-m", "gpu", "-k",
                        "exact_integers", "-p", "no:cacheprovider"], env=e, capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert f"{len(SHAPES)} passed" in r.stdout

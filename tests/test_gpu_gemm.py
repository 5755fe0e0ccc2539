"""GPU: the tcgen05 grouped GEMM through the C-ABI test hook.

Inputs on the 5-bit dyadic grid make every fp32 accumulation exact, so the fp32
epilogue must equal the fp64 reference BIT-EXACTLY (any indexing/descriptor/
swizzle bug shows up as a mismatch).  SwiGLU / SiLU epilogues are compared with
a plain PyTorch fp32 reference within bf16 rounding.
"""
import pytest
import torch

import probe_inputs as pi

pytestmark = pytest.mark.gpu


def _grid(shape, seed):
    return pi.dyadic(shape, "gemm-test", seed, device="cuda")


def _ref(A, B, groups, N):
    out = {}
    for (a_row, m, b_row, c_row) in groups:
        out[c_row] = (A[a_row:a_row + m].double() @ B[b_row:b_row + N].double().T)
    return out


@pytest.mark.parametrize("mode,N,K", [(0, 256, 256), (0, 136, 720), (2, 384, 512), (2, 256, 2048)])
def test_gemm_f32_exact(mode, N, K):
    from paper_2602_00509_b200 import test_gemm
    A = _grid((700, K), 1 + K)
    B = _grid((4 * N, K), 2 + K)
    groups = [[0, 300, 0, 0], [300, 1, N, 300], [301, 0, 2 * N, 301], [310, 389, 3 * N, 301]]
    Cout = torch.full((700, N), float("nan"), device="cuda")
    test_gemm(A, B, groups, N, mode, Cout)
    torch.cuda.synchronize()
    ref = _ref(A, B, groups, N)
    for (a_row, m, b_row, c_row) in groups:
        if m == 0:
            continue
        got = Cout[c_row:c_row + m].double()
        assert torch.equal(got, ref[c_row]), (mode, N, K, a_row, (got - ref[c_row]).abs().max())


def test_gemm_swiglu_and_silu():
    from paper_2602_00509_b200 import test_gemm
    F, K = 384, 512
    A = (torch.randn(333, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(2 * (2 * F), K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    groups = [[0, 200, 0, 0], [200, 133, 2 * F, 200]]
    act = torch.zeros(333, F, dtype=torch.bfloat16, device="cuda")
    test_gemm(A, B, groups, 2 * F, 1, act)
    torch.cuda.synchronize()
    for (a_row, m, b_row, c_row) in groups:
        g = A[a_row:a_row + m].float() @ B[b_row:b_row + F].float().T
        u = A[a_row:a_row + m].float() @ B[b_row + F:b_row + 2 * F].float().T
        ref = torch.nn.functional.silu(g) * u
        got = act[c_row:c_row + m].float()
        err = (got - ref).abs().max().item()
        assert err <= 2 ** -7 * ref.abs().max().item() + 1e-3, err
    # SiLU → bf16 epilogue (predictor residual activation)
    out = torch.zeros(333, 256, dtype=torch.bfloat16, device="cuda")
    test_gemm(A, B[:256], [[0, 333, 0, 0]], 256, 3, out)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(A.float() @ B[:256].float().T)
    assert (out.float() - ref).abs().max().item() <= 2 ** -7 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("mode,N,K,rows,variant", [(0, 256, 256, 40000, 0), (2, 512, 768, 30000, 1),
                                                   (2, 512, 768, 30000, 10), (0, 128, 2048, 65536, 0),
                                                   (0, 384, 512, 20000, 11), (2, 2048, 768, 9000, 10),
                                                   (2, 512, 768, 30000, 6), (2, 2048, 768, 9000, 6),
                                                   (2, 256, 2048, 700, 6), (0, 128, 2560, 30000, 11),
                                                   (0, 128, 2560, 30000, 12), (2, 136, 640, 9001, 12)])
def test_gemm_multi_tile_per_cta_exact(mode, N, K, rows, variant):
    """Several tiles per persistent CTA (TMEM accumulator double buffer, phase wrap-around),
    every kernel variant (BN, stages, epilogue warps)."""
    from paper_2602_00509_b200 import bench_gemm
    A = _grid((rows, K), 11 + K)
    B = _grid((2 * N, K), 12 + K)
    half = rows // 2 + 77
    groups = [[0, half, 0, 0], [half, rows - half, N, half]]
    Cout = torch.full((rows, N), float("nan"), device="cuda")
    bench_gemm(A, B, groups, N, mode, Cout, variant=variant, reps=1)
    torch.cuda.synchronize()
    ref = _ref(A, B, groups, N)
    for (a_row, m, b_row, c_row) in groups:
        got = Cout[c_row:c_row + m].double()
        bad = (got != ref[c_row]).any(dim=1).nonzero()
        assert bad.numel() == 0, (mode, N, K, rows, bad[:10].flatten().tolist())


@pytest.mark.parametrize("variant", [1, 6, 10, 13])
def test_gemm_multi_tile_swiglu(variant):
    from paper_2602_00509_b200 import bench_gemm
    F, K, rows = 768, 2048, 20000
    A = _grid((rows, K), 21)
    B = _grid((2 * F, K), 22)
    act = torch.zeros(rows, F, dtype=torch.bfloat16, device="cuda")
    bench_gemm(A, B, [[0, rows, 0, 0]], 2 * F, 1, act, variant=variant, reps=1)
    torch.cuda.synchronize()
    g = A.double() @ B[:F].double().T
    u = A.double() @ B[F:].double().T
    ref = (torch.nn.functional.silu(g) * u)
    err = ((act.double() - ref).abs() / (ref.abs() + 1e-3)).max().item()
    assert err < 2 ** -7, err


@pytest.mark.parametrize("N,K,rows,variant", [(256, 256, 3000, 0), (2048, 768, 9000, 10), (2048, 768, 9000, 6),
                                              (512, 768, 30000, 6), (2880, 640, 1000, 6), (2880, 640, 1000, 10),
                                              (2048, 768, 9000, 13), (2880, 640, 1000, 13), (512, 768, 30000, 13),
                                              (2048, 768, 9000, 14), (2880, 640, 1000, 14)])
def test_gemm_f16_output_exact(N, K, rows, variant):
    """The expert-output epilogue (fp16 Y, D2): TMA tensor stores in SWIZZLE_64B for full
    32-row slabs, masked row stores for group tails.  Dyadic inputs make the fp32
    accumulator exact, so the fp16 output must equal round-to-nearest-even of the exact
    product (torch's fp64 → fp16 conversion) bit-for-bit."""
    from paper_2602_00509_b200 import bench_gemm
    A = _grid((rows, K), 31 + K)
    B = _grid((2 * N, K), 32 + K)
    half = rows // 2 + 77
    groups = [[0, half, 0, 0], [half, rows - half, N, half]]
    Cout = torch.full((rows, N), float("nan"), dtype=torch.float16, device="cuda")
    bench_gemm(A, B, groups, N, 7, Cout, variant=variant, reps=1)
    torch.cuda.synchronize()
    ref = _ref(A, B, groups, N)
    for (a_row, m, b_row, c_row) in groups:
        exp = ref[c_row].to(torch.float16)
        got = Cout[c_row:c_row + m]
        bad = (got.view(torch.int16) != exp.view(torch.int16)).any(dim=1).nonzero()
        assert bad.numel() == 0, (N, K, rows, variant, bad[:10].flatten().tolist())

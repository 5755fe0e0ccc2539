"""Time grouped-GEMM kernel variants on the C1 expert shapes (isolated, CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_00509_b200 import bench_gemm  # noqa: E402

torch.manual_seed(0)
E_loc, rows_per = 128, 4096          # C1 whole EP group on one GPU: 128 experts × 4096 rows (balanced)
H, F = 2048, 768
M = E_loc * rows_per
res = {}
# GEMM2: act [M, F] × W2 [E·H, F]^T → Y fp32 [M, H]
A = (torch.randn(M, F, device="cuda") * 0.5).to(torch.bfloat16)
B = (torch.randn(E_loc * H, F, device="cuda") / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(M, H, device="cuda")
groups = [[e * rows_per, rows_per, e * H, e * rows_per] for e in range(E_loc)]
fl = 2.0 * M * H * F
for v in (1, 2):
    ms = bench_gemm(A, B, groups, H, 2, Y, variant=v, reps=10)
    res[f"gemm2_v{v}"] = {"ms": ms, "tflops": fl / ms / 1e9}
del A, B, Y
# GEMM1: recv [M, H] × W13 [E·2F, H]^T → SwiGLU act bf16 [M, F]
A = (torch.randn(M, H, device="cuda") * 0.5).to(torch.bfloat16)
B = (torch.randn(E_loc * 2 * F, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
groups = [[e * rows_per, rows_per, e * 2 * F, e * rows_per] for e in range(E_loc)]
fl = 4.0 * M * H * F
for v in (1, 2):
    ms = bench_gemm(A, B, groups, 2 * F, 1, act, variant=v, reps=10)
    res[f"gemm1_v{v}"] = {"ms": ms, "tflops": fl / ms / 1e9}
print(json.dumps(res))

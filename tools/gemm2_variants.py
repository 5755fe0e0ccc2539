"""Interleaved best-of-N timing of expert GEMM2 (fp16 Y, mode 7) and GEMM1 (SwiGLU, mode 1)
kernel variants at C1 shapes (128 local experts × 4096 rows)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_00509_b200 import bench_gemm  # noqa: E402

torch.manual_seed(0)
E_loc, rows_per, H, F = 128, 4096, 2048, 768
M = E_loc * rows_per
A2 = (torch.randn(M, F, device="cuda") * 0.5).to(torch.bfloat16)
B2 = (torch.randn(E_loc * H, F, device="cuda") / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(M, H, dtype=torch.float16, device="cuda")
g2 = [[e * rows_per, rows_per, e * H, e * rows_per] for e in range(E_loc)]
A1 = (torch.randn(M, H, device="cuda") * 0.5).to(torch.bfloat16)
B1 = (torch.randn(E_loc * 2 * F, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
g1 = [[e * rows_per, rows_per, e * 2 * F, e * rows_per] for e in range(E_loc)]
variants = [int(v) for v in sys.argv[1:]] or [6, 7]
res = {}
for rnd in range(4):
    for v in variants:
        ms = bench_gemm(A2, B2, g2, H, 7, Y, variant=v, reps=5)
        res.setdefault(f"gemm2_f16_v{v}", []).append(round(2.0 * M * H * F / ms / 1e9, 1))
        ms = bench_gemm(A1, B1, g1, 2 * F, 1, act, variant=v, reps=5)
        res.setdefault(f"gemm1_v{v}", []).append(round(4.0 * M * H * F / ms / 1e9, 1))
print(json.dumps({k: {"best": max(v), "all": v} for k, v in res.items()}))

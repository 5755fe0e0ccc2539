"""Time grouped-GEMM kernel variants on the C1 expert shapes (isolated, CUDA events).
mode 2 = fp32 store, mode 4 = TMEM read but no global stores (epilogue-bound test)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_00509_b200 import bench_gemm  # noqa: E402

torch.manual_seed(0)
E_loc, rows_per = 128, 4096
H, F = 2048, 768
M = E_loc * rows_per
res = {}
A = (torch.randn(M, F, device="cuda") * 0.5).to(torch.bfloat16)
B = (torch.randn(E_loc * H, F, device="cuda") / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(M, H, device="cuda")
groups = [[e * rows_per, rows_per, e * H, e * rows_per] for e in range(E_loc)]
fl = 2.0 * M * H * F
for mode in (2, 4):
    for v in (1, 2):
        ms = bench_gemm(A, B, groups, H, mode, Y, variant=v, reps=10)
        res[f"gemm2_mode{mode}_v{v}"] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}
print(json.dumps(res))

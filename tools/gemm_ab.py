"""Expert-GEMM shapes of the C1 layer through the C-ABI timing hook (probe_bench_gemm):
GEMM2 (K = F = 768, N = H = 2048, fp16 Y) on the CTA-pair 256×256 kernel (variant 6) and the
256×512 one-accumulator kernel (variant 13; 14 with double-buffered stores), and GEMM1 (K = H = 2048, SwiGLU over 2F = 1536 →
bf16 act, variants 6 and 13), on 137 uniform groups of the C1 layer's total rows.  PROBE_LIB_PATH
selects the library build (A/B of two builds).  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_00509_b200 import bench_gemm  # noqa: E402

dev = "cuda"
H, F, rows, ng, slots = 2048, 768, 524288, 137, 152
per = rows // ng
groups2 = [[i * per, per, (i % slots) * H, i * per] for i in range(ng)]
A2 = (torch.randn(rows, F, device=dev) * 0.5).to(torch.bfloat16)
B2 = (torch.randn(slots * H, F, device=dev) / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(rows, H, dtype=torch.float16, device=dev)
out = {"lib": os.environ.get("PROBE_LIB_PATH", "in-tree")}
for rep in range(3):
    for v in (6, 13, 14):
        ms2 = bench_gemm(A2, B2, groups2, H, 7, Y, variant=v, reps=10)        # mode 7: EPI_F16
        out.setdefault(f"gemm2_v{v}_TFs", []).append(round(2.0 * per * ng * H * F / ms2 / 1e9, 1))
del A2, B2, Y
A1 = (torch.randn(rows, H, device=dev) * 0.5).to(torch.bfloat16)
B1 = (torch.randn(slots * 2 * F, H, device=dev) / H ** 0.5).to(torch.bfloat16)
act = torch.empty(rows, F, dtype=torch.bfloat16, device=dev)
groups1 = [[i * per, per, (i % slots) * 2 * F, i * per] for i in range(ng)]
for rep in range(3):
    for v in (6, 13):
        ms1 = bench_gemm(A1, B1, groups1, 2 * F, 1, act, variant=v, reps=10)  # mode 1: EPI_SWIGLU
        out.setdefault(f"gemm1_v{v}_TFs", []).append(round(4.0 * per * ng * H * F / ms1 / 1e9, 1))
print(json.dumps(out))

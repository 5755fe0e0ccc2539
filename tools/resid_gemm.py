"""Small-N GEMM shapes of the predictor / gate through the timing hook (grid = all SMs):
the fused predictor's residual a·Ŵ2ᵀ (M = 65536, K = h = 512, N = E = 128) and the router GEMM
(K = H = 2048, N = 128), by variant and epilogue mode.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_00509_b200 import bench_gemm  # noqa: E402

dev = "cuda"
M = 65536
res = {}
for name, K in (("resid_K512", 512), ("gate_K2048", 2048)):
    A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    B = (torch.randn(128, K, device=dev) / K ** 0.5).to(torch.bfloat16)
    C = torch.empty(M, 128, device=dev)
    for v in (0, 12):
        for mode in (0, 4):
            ms = bench_gemm(A, B, [[0, M, 0, 0]], 128, mode, C, variant=v, reps=20)
            res[f"{name}_v{v}_mode{mode}_us"] = round(ms * 1e3, 1)
print(json.dumps(res))

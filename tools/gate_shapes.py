"""Isolated timing of the BN=128 GEMM shapes of the gate and the predictor (C1, 8 ranks)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2602_00509_b200 import bench_gemm
M, H, E, h = 65536, 2048, 128, 512
x = (torch.randn(M, H, device="cuda") * 0.3).to(torch.bfloat16)
W = (torch.randn(512, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
res = {}
C32 = torch.empty(M, 512, device="cuda")
Cb = torch.empty(M, 512, dtype=torch.bfloat16, device="cuda")
ids = torch.empty(M, 8, dtype=torch.int32, device="cuda")
g = [[0, M, 0, 0]]
for name, mode, N, out, v in [("gate_f32_N128", 0, 128, C32, 0), ("gate_topk_N128", 5, 128, ids, 0),
                              ("pred_count_N128", 6, 128, ids, 0), ("silu_N512_bn128", 3, 512, Cb, 0),
                              ("silu_N512_bn256", 3, 512, Cb, 1), ("f32_N512_bn128", 0, 512, C32, 0),
                              ("none_N128", 4, 128, C32, 0)]:
    ms = bench_gemm(x, W, g, N, mode, out, variant=v, reps=20)
    res[name] = {"us": round(ms * 1e3, 1), "tflops": round(2.0 * M * H * N / ms / 1e9, 1),
                 "x_read_TBps": round(M * H * 2 / ms / 1e9, 2)}
print(json.dumps(res))

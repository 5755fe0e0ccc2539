"""Per-role wait-cycle breakdown of the expert GEMMs (C1 shapes) using the analysis build
tools/libprobe_stats.so (nvcc ... -DPROBE_GEMM_STATS).  Prints the library's [gemm stats]
lines (stderr): producer waits on `empty`, MMA waits on `full` / `tempty`, epilogue waits
on `tfull` and busy cycles, summed over CTAs."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_00509_b200 import _lib  # noqa: E402

os.environ["PROBE_GEMM_STATS"] = "1"
lib = C.CDLL("tools/libprobe_stats.so")
lib.probe_bench_gemm.restype = C.c_int32
lib.probe_bench_gemm.argtypes = _lib.load().probe_bench_gemm.argtypes
E_loc, rows_per, H, F = 128, 4096, 2048, 768
M = E_loc * rows_per


def run(A, B, groups, N, mode, out, v):
    flat = (C.c_int32 * (4 * len(groups)))(*[int(x) for g in groups for x in g])
    ms = C.c_float(0)
    st = lib.probe_bench_gemm(C.c_void_p(A.data_ptr()), A.shape[0], C.c_void_p(B.data_ptr()), B.shape[0], A.shape[1],
                              N, flat, len(groups), mode, v, 5, C.byref(ms), C.c_void_p(out.data_ptr()),
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    return ms.value


V = int(sys.argv[1]) if len(sys.argv) > 1 else 6     # 6: CTA-pair <256,6,4> (product default)
Y = torch.empty(M, H, device="cuda")
g2 = [[e * rows_per, rows_per, e * H, e * rows_per] for e in range(E_loc)]
for K in (768, 1536, 2048):   # GEMM2 is K = F = 768; longer K isolates the per-tile cost
    A2 = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B2 = (torch.randn(E_loc * H, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    for mode in (7, 4):      # fp16 Y (product), no stores
        ms = run(A2, B2, g2, H, mode, Y, V)
        print("GEMM2-shape K", K, "mode", mode, "ms", ms, "TF/s", round(2.0 * M * H * K / ms / 1e9, 1), flush=True)
    del A2, B2
# one group of all rows (no group boundaries / ragged tiles)
A2 = (torch.randn(M, F, device="cuda") * 0.5).to(torch.bfloat16)
B2 = (torch.randn(H, F, device="cuda") / F ** 0.5).to(torch.bfloat16)
ms = run(A2, B2, [[0, M, 0, 0]], H, 7, Y, V)
print("GEMM2 one group ms", ms, "TF/s", round(2.0 * M * H * F / ms / 1e9, 1), flush=True)
del A2, B2, Y
A1 = (torch.randn(M, H, device="cuda") * 0.5).to(torch.bfloat16)
B1 = (torch.randn(E_loc * 2 * F, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
g1 = [[e * rows_per, rows_per, e * 2 * F, e * rows_per] for e in range(E_loc)]
ms = run(A1, B1, g1, 2 * F, 1, act, V)
print("GEMM1 ms", ms, "TF/s", round(4.0 * M * H * F / ms / 1e9, 1), flush=True)
del A1, B1, act
# predictor Ŵ1·x shape (C1: M = 65536 tokens, N = h = 512, K = H = 2048): SiLU→bf16 (mode 3,
# manual stores), no store (4), fp32 TMA stores (0); 1-CTA <128,6,4> (0) and CTA pairs (6)
Mp, Np, Kp = 65536, 512, 2048
Ap = (torch.randn(Mp, Kp, device="cuda") * 0.5).to(torch.bfloat16)
Bp = (torch.randn(Np, Kp, device="cuda") / Kp ** 0.5).to(torch.bfloat16)
Cp = torch.empty(Mp, Np, device="cuda")
for v in (0, 6):
    for mode in (3, 4, 0):
        ms = run(Ap, Bp, [[0, Mp, 0, 0]], Np, mode, Cp, v)
        print("predictor W1x variant", v, "mode", mode, "ms", ms, "TF/s", round(2.0 * Mp * Np * Kp / ms / 1e9, 1),
              flush=True)

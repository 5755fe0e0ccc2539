"""A/B the grouped GEMM of two builds of libprobe.so on the same box (isolated, CUDA events).
usage: python tools/ab_gemm.py [other.so ...]   (the in-tree library is always 'cur')"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_00509_b200 import _lib  # noqa: E402


def bench(lib, A, B, groups, N, mode, out, variant, reps):
    flat = (C.c_int32 * (4 * len(groups)))(*[int(v) for g in groups for v in g])
    ms = C.c_float(0)
    st = lib.probe_bench_gemm(C.c_void_p(A.data_ptr()), A.shape[0], C.c_void_p(B.data_ptr()), B.shape[0],
                              A.shape[1], N, flat, len(groups), mode, variant, reps, C.byref(ms),
                              C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return ms.value if st == 0 else None


libs = {"cur": _lib.load()}
for p in sys.argv[1:]:
    l = C.CDLL(p)
    l.probe_bench_gemm.restype = C.c_int32
    l.probe_bench_gemm.argtypes = _lib.load().probe_bench_gemm.argtypes
    libs[p.split("/")[-1]] = l
torch.manual_seed(0)
E_loc, rows_per, H, F = 128, 4096, 2048, 768
M = E_loc * rows_per
res = {}
A2 = (torch.randn(M, F, device="cuda") * 0.5).to(torch.bfloat16)
B2 = (torch.randn(E_loc * H, F, device="cuda") / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(M, H, dtype=torch.float16, device="cuda")   # fp16 Y (mode 7)
g2 = [[e * rows_per, rows_per, e * H, e * rows_per] for e in range(E_loc)]
A1 = (torch.randn(M, H, device="cuda") * 0.5).to(torch.bfloat16)
B1 = (torch.randn(E_loc * 2 * F, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
g1 = [[e * rows_per, rows_per, e * 2 * F, e * rows_per] for e in range(E_loc)]
for rnd in range(3):
    for name, lib in libs.items():
        for v in (6, 7):
            ms = bench(lib, A2, B2, g2, H, 7, Y, v, 20)
            if ms is None:
                continue
            res.setdefault(f"{name}/gemm2_f16_v{v}", []).append(round(2.0 * M * H * F / ms / 1e9, 1))
            ms = bench(lib, A1, B1, g1, 2 * F, 1, act, v, 20)
            res.setdefault(f"{name}/gemm1_v{v}", []).append(round(4.0 * M * H * F / ms / 1e9, 1))
print(json.dumps(res))

import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2602_00509_b200 import bench_gemm
rows, N, K = 64, 128, 64
A = torch.zeros(rows, K, device="cuda"); B = torch.zeros(N, K, device="cuda")
# A[r, 0] = r, B[n, 0] = 1 and B[n,1]=n/256 with A[r,1]=1 -> C[r,n] = r + n/256 (exact in fp16 for small)
A[:, 0] = torch.arange(rows, device="cuda").float(); A[:, 1] = 1.0
B[:, 0] = 1.0; B[:, 1] = torch.arange(N, device="cuda").float() / 128
A = A.to(torch.bfloat16); B = B.to(torch.bfloat16)
for groups in ([[0, 64, 0, 0]], [[0, 40, 0, 0]]):
    C = torch.full((rows, N), float("nan"), dtype=torch.float16, device="cuda")
    bench_gemm(A, B, groups, N, 7, C, variant=0, reps=1); torch.cuda.synchronize()
    m = groups[0][1]
    exp = (A.float() @ B.float().T)[:m].half()
    got = C[:m]
    bad = (got != exp)
    print("groups", groups, "bad", int(bad.sum()), "of", bad.numel())
    if bad.any():
        idx = bad.nonzero()[:12].tolist()
        for r, c in idx: print(r, c, float(got[r, c]), float(exp[r, c]))

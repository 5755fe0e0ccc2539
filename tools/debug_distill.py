import sys, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_distill import _setup, CASES
sh, T = CASES["mid-ragged"]
rt, x, xn, W, b, w1, w2 = _setup(sh, 2, zero_w2=True, same_x=True)
N = sh.G * T
g1 = torch.empty(sh.h, sh.H, device="cuda"); g2 = torch.empty(sh.E, sh.h, device="cuda")
stats = torch.empty(4, dtype=torch.float64, device="cuda")
sl = torch.empty(N, sh.E, device="cuda"); tl = torch.empty(N, sh.E, device="cuda")
rt.distill_grad(x, xn, W, b, w1, w2, g1, g2, stats, sl, tl)
torch.cuda.synchronize()
d = (sl - tl)
print("max |sl-tl|", d.abs().max().item(), "nonzero", torch.count_nonzero(d).item(), "of", d.numel())
idx = torch.nonzero(d)[:5]
for i in idx.tolist():
    print(i, sl[i[0], i[1]].item(), tl[i[0], i[1]].item())
print("stats", stats.tolist())
ref = (x.reshape(N, -1).float() @ W.float().T)
print("max |tl-ref|", (tl - ref).abs().max().item(), "max|sl-ref|", (sl - ref).abs().max().item())

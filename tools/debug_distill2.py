import sys, math, torch
sys.path.insert(0, ".")
import probe_inputs as pi
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
from paper_2602_00509_b200.distill import PredictorDistiller, metrics
sh = pi.SHAPES[sys.argv[1]].with_(T=int(sys.argv[2]))
held = pi.distill_task(sh, 1000, device="cuda")
tr = pi.distill_task(sh, 0, device="cuda")
N = sh.G * sh.T
rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=64, T=sh.T, h=sh.h))
w1 = (torch.randn(sh.h, sh.H) / math.sqrt(sh.H)).to(torch.bfloat16).cuda()
w2 = torch.zeros(sh.E, sh.h, dtype=torch.bfloat16, device="cuda")
d = PredictorDistiller(rt, w1, w2)
for i in range(3):
    d.grad(held.x, held.x_next, held.W); print("eval", i, metrics(d.stats, N, sh.k), flush=True)
for i in range(3):
    m = d.step(tr.x, tr.x_next, tr.W, lr=4.0); print("step", i, m, d.g1.abs().max().item(), d.g2.abs().max().item(), d.m2.abs().max().item(), flush=True)
    d.grad(held.x, held.x_next, held.W); print("eval", metrics(d.stats, N, sh.k), flush=True)
rt.check()

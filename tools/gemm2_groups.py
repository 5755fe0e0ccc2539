"""Is expert GEMM2's in-layer rate (≈0.68 of sustained vs ≈0.80 isolated) a property of the
layer's group structure?  Take the group sizes of a real C1 layer (8 logical ranks, Zipf 1.0,
plan with replicas; probe_debug_layout), lay the groups out as GEMM2 sees them (rank r's
receive rows from r·cap, local slots in order), and time the same grouped GEMM
(K = F = 768, N = H = 2048, fp16 Y) through the C-ABI test hook against uniform groups with
the same total rows.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import probe_inputs as pi  # noqa: E402
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime, bench_gemm  # noqa: E402
from paper_2602_00509_b200.costs import cost_model, window_ns  # noqa: E402

sh = pi.C1
G, E, k, H, F, T = sh.G, sh.E, sh.k, sh.H, sh.F, sh.T
a, b, n, bw = cost_model(H, F)
cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=F, T=T, h=sh.h, alpha_ps=a, beta_ps=b, n_sat=n, bw_bytes_per_us=bw,
                  capacity_factor=4.0)
rt = ProbeRuntime(cfg)
dev = "cuda"
L = [pi.layer_inputs(sh, 0, i, 1.0, device=dev) for i in (0, 1)]
W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
ex = [pi.expert_weights(sh, p, device=dev) for p in (0, 1)]
res = pi.predictor_residual(sh, 1, device=dev)
out = torch.empty(G, T, H, device=dev)
win = torch.full((G,), window_ns(H, F, T, k, E=E, G=G), dtype=torch.int64, device=dev)
rt.forward(0, L[0].x, W[0], None, ex[0][0], ex[0][1], out)
rt.predict(1, L[0].x, W[1], None, res[0], res[1])
rt.plan(1, win)
rt.prefetch(1, ex[1][0], ex[1][1], phase=0)
rt.forward(1, L[1].x, W[1], None, ex[1][0], ex[1][1], out, use_plan=True)
S = E // G + 3
rows = torch.empty(G, S, dtype=torch.int32, device=dev)
rt.debug_layout(group_rows=rows)
torch.cuda.synchronize()
rows = rows.cpu().tolist()
cap = cfg.recv_capacity
rt.close()
del L, ex, out
torch.cuda.empty_cache()
groups, slot_w = [], 0
for r in range(G):
    off = r * cap
    for j in range(S):
        m = rows[r][j]
        if m > 0:
            groups.append([off, m, slot_w * H, off])
        off += m
        slot_w += 1
A = (torch.randn(G * cap, F, device=dev) * 0.5).to(torch.bfloat16)
B = (torch.randn(slot_w * H, F, device=dev) / F ** 0.5).to(torch.bfloat16)
Y = torch.empty(G * cap, H, dtype=torch.float16, device=dev)
tot = sum(g[1] for g in groups)
ms_layer = bench_gemm(A, B, groups, H, 7, Y, variant=6, reps=10)
ng = len(groups)
uni, per = [], tot // ng
for i in range(ng):
    m = per if i < ng - 1 else tot - per * (ng - 1)
    uni.append([i * per, m, (i % slot_w) * H, i * per])
ms_uni = bench_gemm(A, B, uni, H, 7, Y, variant=6, reps=10)
fl = 2.0 * tot * H * F
print(json.dumps({"groups": ng, "rows": tot, "max_group": max(g[1] for g in groups),
                  "min_group": min(g[1] for g in groups),
                  "layer_groups_ms": ms_layer, "layer_groups_TFs": fl / ms_layer / 1e9,
                  "uniform_groups_ms": ms_uni, "uniform_groups_TFs": fl / ms_uni / 1e9}))

import os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import probe_inputs as pi
import oracle as O
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
sh = pi.C0
cfg = ProbeConfig(G=2, E=8, k=2, H=256, F=512, T=64, h=64)
rt = ProbeRuntime(cfg)
W = pi.router_weight(sh, 0, device="cuda")
w13, w2 = pi.expert_weights(sh, 0, device="cuda")
out = torch.empty(2, 64, 256, device="cuda")
ids = torch.empty(2, 64, 2, dtype=torch.int32, device="cuda")
bad_total = 0
for step in range(6):
    li = pi.layer_inputs(sh, step, 0, 1.5, device="cuda")
    ref = [O.gate(pi.bf16_to_numpy_f64(li.x[r]), pi.bf16_to_numpy_f64(W), None, 2)[0] for r in range(2)]
    for rep in range(5):
        rt.forward(0, li.x, W, None, w13, w2, out, topk_ids=ids)
        torch.cuda.synchronize()
        a = ids.cpu().numpy()
        for r in range(2):
            bad = np.nonzero((a[r] != ref[r]).any(axis=1))[0]
            if len(bad):
                bad_total += len(bad)
                print(os.environ.get("PROBE_UNFUSED"), step, rep, r, bad[:4], a[r][bad[:2]].tolist(), ref[r][bad[:2]].tolist())
print("bad_total", bad_total)

"""Robustness to an abrupt hotspot shift (the shape of PAPER.md Fig. `fig:robustness`,
P:553-567), on one B200 with the EP straggler emulation (expert GEMMs partitioned per
logical rank, PROBE_OPT_EP_EMULATION).  Policies, all on the same library kernels:
  static  — static EP, no replication;
  probe   — PROBE: lookahead predictor + planner + split-phase prefetch every layer;
  eplb    — statistics-based one-shot policy: accumulate the actual
            counts of the first W layers, plan once from that history, keep re-using it.
Phase A: hotspot permutation A for N_A layers; phase B: permutation B for N_B layers.
Per-layer main-stream latency from the library's CUDA-event profile.
usage: python tools/robustness.py [--T 8192] [--zipf 1.0]"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import probe_inputs as pi  # noqa: E402
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime  # noqa: E402
from paper_2602_00509_b200._lib import PHASES  # noqa: E402
from paper_2602_00509_b200._lib import OPT_EP_EMULATION  # noqa: E402
from paper_2602_00509_b200.costs import cost_model, window_ns  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=8192)
ap.add_argument("--zipf", type=float, default=1.0)
ap.add_argument("--layers-a", type=int, default=24)
ap.add_argument("--layers-b", type=int, default=24)
ap.add_argument("--history", type=int, default=8)
args = ap.parse_args()

shape = pi.C1.with_(T=args.T)
G, E, k, H, F, T = shape.G, shape.E, shape.k, shape.H, shape.F, shape.T
a, b, n, bw = cost_model(H, F)
# PROBE: 3 redundant experts per rank; the statistics-based one-shot policy is configured
# as the paper's EPLB baseline, 2 redundant expert slots per layer per rank
rts = {}
for name, budget in (("probe", 3), ("eplb", 2)):
    cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=F, T=T, h=shape.h, n_sat=n, alpha_ps=a, beta_ps=b,
                      bw_bytes_per_us=bw, capacity_factor=4.0, replica_budget=budget)
    rts[name] = ProbeRuntime(cfg)
    rts[name].set_option(OPT_EP_EMULATION, 1)
dev = "cuda"
POOL = 4
pools = {ph: [pi.layer_inputs(shape, 0, i, args.zipf, device=dev, wrap=POOL, perm_key=key) for i in range(POOL)]
         for ph, key in (("A", 1001), ("B", 2002))}
W = [pi.router_weight(shape, p, device=dev) for p in (0, 1)]
ex = [pi.expert_weights(shape, p, device=dev) for p in (0, 1)]
res = [pi.predictor_residual(shape, p, device=dev) for p in (0, 1)]
win = torch.full((G,), window_ns(H, F, T, k, E=E, G=G), dtype=torch.int64, device=dev)
out = torch.empty(G, T, H, device=dev)
hist = [torch.zeros(G, E, dtype=torch.int32, device=dev) for _ in (0, 1)]


def run(policy):
    rt = rts["eplb" if policy == "eplb" else "probe"]
    seq = ["A"] * args.layers_a + ["B"] * args.layers_b
    rt.profile(len(seq))
    planned = False
    for L, ph in enumerate(seq):
        x = pools[ph][L % POOL].x
        p, q = L % 2, (L + 1) % 2
        rt.forward(L, x, W[p], None, ex[p][0], ex[p][1], out, use_plan=planned)
        planned = False
        if policy == "probe":
            rt.predict(L + 1, x, W[q], None, res[q][0], res[q][1])
            rt.plan(L + 1, win)
            rt.prefetch(L + 1, ex[q][0], ex[q][1], phase=0)
            planned = True
        elif policy == "eplb":
            if L < args.history:
                rt.history_update(L, hist[p], reset=(L < 2))
            else:
                rt.plan(L + 1, win, pred_counts=hist[q])
                rt.prefetch(L + 1, ex[q][0], ex[q][1], phase=0)
                planned = True
    ms = rt.profile_read()[:, PHASES.index("total")].numpy()
    na = args.layers_a
    skip = max(args.history + 2, 4)
    return {"phase_A_ms": float(np.mean(ms[skip:na])), "phase_B_ms": float(np.mean(ms[na + 2:])),
            "per_layer_ms": [round(float(v), 3) for v in ms]}


result = {}
for policy in ("static", "probe", "eplb"):
    run(policy)                      # warm-up pass (clocks, caches)
    result[policy] = run(policy)
result["config"] = {"shape": "C1", "T": T, "G": G, "zipf": args.zipf, "layers_a": args.layers_a,
                    "layers_b": args.layers_b, "history_layers": args.history,
                    "replica_budget": {"probe": 3, "eplb": 2},
                    "note": "EP straggler emulation on one B200; hotspot permutation A then B"}
print(json.dumps(result))

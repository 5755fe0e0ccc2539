"""Device-detected failures (include/probe.h, SURVEY §8(b) "Errors"), driven on the GPU.

1. A plan built from a badly wrong prediction would overflow a rank's receive capacity on
   the ACTUAL counts: the layout kernel falls back to static EP for that layer, on device
   and identically on every rank (probe_debug_flags word 4 counts it); the layer output is
   the same function (semantic equivalence), so it still matches the oracle's
   static-EP layer within 2e-2·RMS and the dispatch route is bit-exactly static EP.
2. Static EP itself overflows (capacity below the hottest rank's rows under heavy skew):
   the device error word is raised and probe_check returns PROBE_ECAPACITY.
"""
import numpy as np
import pytest
import torch

import oracle as O
import probe_inputs as pi
from layer_harness import f64

pytestmark = pytest.mark.gpu

SH = pi.C0.with_(name="fail", E=16, k=2, H=256, F=128, T=128, G=4)


def _inputs(zipf_s):
    dev = "cuda"
    li0 = pi.layer_inputs(SH, 0, 0, zipf_s, device=dev)
    li1 = pi.layer_inputs(SH, 0, 1, zipf_s, device=dev)
    W = [pi.router_weight(SH, p, device=dev) for p in (0, 1)]
    w = [pi.expert_weights(SH, p, device=dev) for p in (0, 1)]
    return li0, li1, W, w


def _static_rows(x, W):
    G, E, EL = SH.G, SH.E, SH.E // SH.G
    ref = O.layer_reference([f64(x[r]) for r in range(G)], f64(W), None, SH.k, None, G, E)
    return ref, [sum(ref["layout"].group_sizes[r]) for r in range(G)]


def test_plan_overflow_falls_back_to_static_ep():
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    G, E, EL = SH.G, SH.E, SH.E // SH.G
    li0, li1, W, w = _inputs(1.3)
    ref1, rows = _static_rows(li1.x, W[1])
    hot = int(np.argmax(rows))
    donor = (hot + 1) % G
    # misprediction: the donor rank's experts look hot and the (actually hottest) rank idle,
    # so the planner replicates donor experts ONTO the hottest rank
    nhat = np.full((G, E), 4, dtype=np.int64)
    nhat[:, donor * EL:(donor + 1) * EL] = 60
    nhat[:, hot * EL:(hot + 1) * EL] = 0
    pcfg = O.PlannerConfig(G=G, E=E, replica_budget=3, kmax=16, alpha_ps=1, beta_ps=0, n_sat=0,
                           bw_bytes_per_us=770_000, expert_bytes=3 * SH.H * SH.F * 2)
    plan = O.plan_greedy(nhat, [10 ** 9] * G, pcfg)
    assert plan.replicas[hot], "test design: the plan must replicate onto the hottest rank"
    n = ref1["n"]
    split = O.materialize(n, plan.quota, plan.replicas, G, E)
    planned = [int(split[:, :, r].sum()) for r in range(G)]
    cap = (max(rows) + 7) // 8 * 8                       # recv_capacity is a multiple of 8
    assert planned[hot] > cap, (planned, rows)          # the plan would overflow, static fits
    cfg = ProbeConfig(G=G, E=E, k=SH.k, H=SH.H, F=SH.F, T=SH.T, h=0, recv_capacity=cap)
    rt = ProbeRuntime(cfg)
    out = [torch.empty(G, SH.T, SH.H, device="cuda") for _ in (0, 1)]
    ids = torch.empty(G, SH.T, SH.k, dtype=torch.int32, device="cuda")
    pc = torch.from_numpy(nhat.astype(np.int32)).cuda()
    win = torch.full((G,), 10 ** 9, dtype=torch.int64, device="cuda")
    reps = torch.empty(G, 3, dtype=torch.int32, device="cuda")
    rt.plan(1, win, pred_counts=pc, replicas=reps)
    rt.prefetch(1, w[1][0], w[1][1], phase=0)
    rt.forward(1, li1.x, W[1], None, w[1][0], w[1][1], out[1], use_plan=True, topk_ids=ids)
    fl = rt.flags()
    rt.check()                                           # static EP fits: no error
    assert fl[4] == 1, fl
    exp = np.full((G, 3), -1)
    for r in range(G):
        exp[r, :len(plan.replicas[r])] = plan.replicas[r]
    assert np.array_equal(reps.cpu().numpy(), exp)     # the plan itself is the oracle's
    route = torch.empty(G, SH.T, SH.k, 2, dtype=torch.int32, device="cuda")
    rt.debug_layout(route=route)
    torch.cuda.synchronize()
    ids_np = ids.cpu().numpy()
    for r in range(G):
        assert np.array_equal(route[r, :, :, 0].cpu().numpy(), ids_np[r] // EL)          # static EP
        assert np.array_equal(route[r, :, :, 1].cpu().numpy(), ref1["layout"].row[r])
    W13 = {e: f64(w[1][0][e]) for e in range(E)}
    W2 = {e: f64(w[1][1][e]) for e in range(E)}
    outs = O.moe_outputs_ranks([f64(li1.x[r]) for r in range(G)], ref1["ids"], ref1["g"], W13, W2)
    rms = np.sqrt(np.mean(np.concatenate([o.reshape(-1) for o in outs]) ** 2))
    err = max(np.abs(out[1][r].cpu().numpy() - outs[r]).max() for r in range(G))
    assert err <= 2e-2 * rms, (err, rms)
    rt.close()


def test_static_overflow_raises_ecapacity():
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    from paper_2602_00509_b200._lib import ProbeError
    G = SH.G
    li0, _, W, w = _inputs(1.5)
    _, rows = _static_rows(li0.x, W[0])
    cfg = ProbeConfig(G=G, E=SH.E, k=SH.k, H=SH.H, F=SH.F, T=SH.T, h=0, recv_capacity=(max(rows) - 1) // 8 * 8)
    rt = ProbeRuntime(cfg)
    out = torch.empty(G, SH.T, SH.H, device="cuda")
    rt.forward(0, li0.x, W[0], None, w[0][0], w[0][1], out)
    with pytest.raises(ProbeError, match="CAPACITY"):
        rt.check()
    assert rt.flags()[0] & 1
    rt.close()

"""Split-phase prefetch accounting (a9, R27): whatever the timing split between part 1
(beside the expert GEMMs, until the combine raises the suspend flag) and part 2 (after the
combine), the two parts together push exactly the planned replicas' weights, once each,
and the replica slots then hold the home experts' weights bit-exactly."""
import pytest
import torch

import probe_inputs as pi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("zipf_s", [1.2, 1.5])
def test_prefetch_parts_push_exactly_the_planned_replicas(zipf_s):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    sh = pi.C0.with_(name="pfacct", E=32, k=4, H=512, F=384, T=700, G=4)
    G, E, k, H, F, T = sh.G, sh.E, sh.k, sh.H, sh.F, sh.T
    cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=F, T=T, h=sh.h, replica_budget=3, alpha_ps=1, beta_ps=0, n_sat=0)
    rt = ProbeRuntime(cfg)
    dev = "cuda"
    W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
    ex = [pi.expert_weights(sh, p, device=dev) for p in (0, 1)]
    r1, r2 = pi.predictor_residual(sh, 1, device=dev)
    win = torch.full((G,), 10 ** 9, dtype=torch.int64, device=dev)
    reps = torch.empty(G, 3, dtype=torch.int32, device=dev)
    out = torch.empty(G, T, H, device=dev)
    expert_kib = 3 * H * F * 2 // 1024                       # W13 (2F×H) + W2 (H×F), bf16
    total_reps = 0
    before = rt.prefetch_kib()
    for L in range(4):
        li = pi.layer_inputs(sh, 0, L, zipf_s, device=dev)
        p, q = L % 2, (L + 1) % 2
        rt.forward(L, li.x, W[p], None, ex[p][0], ex[p][1], out, use_plan=L > 0)
        rt.predict(L + 1, li.x, W[q], None, r1, r2)
        rt.plan(L + 1, win, replicas=reps)
        rt.prefetch(L + 1, ex[q][0], ex[q][1], phase=0)
        rt.prefetch(L + 1, phase=1)
        torch.cuda.synchronize()
        rl = reps.cpu()
        total_reps += int((rl >= 0).sum())
        # slots of bank q hold the home experts' weights bit-exactly
        for r in range(G):
            sw13, sw2 = rt.replica_slots(r)
            for s in range(3):
                e = int(rl[r, s])
                if e >= 0:
                    assert torch.equal(sw13[3 * q + s].view(torch.uint8), ex[q][0][e].view(torch.uint8))
                    assert torch.equal(sw2[3 * q + s].view(torch.uint8), ex[q][1][e].view(torch.uint8))
    rt.check()
    after = rt.prefetch_kib()
    pushed = (after[0] - before[0]) + (after[1] - before[1])
    assert total_reps > 0
    assert pushed == total_reps * expert_kib, (after, before, total_reps)
    rt.close()

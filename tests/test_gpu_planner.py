"""GPU: the single-CTA planner kernel (Algorithm 1, R10-R22) bit-exact against the oracle's
greedy on explicit n̂ matrices (random skewed loads, comm term, n_sat knee, window-derived
caps, budgets 0..3), and the statistics-based history hook feeding the same planner."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _rt(G, E, **kw):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    cfg = ProbeConfig(G=G, E=E, k=2, H=256, F=256, T=64, h=64, **kw)
    return ProbeRuntime(cfg), cfg


@pytest.mark.parametrize("seed", range(24))
def test_planner_kernel_matches_oracle(seed):
    r = np.random.default_rng(seed)
    G = int(r.choice([2, 4, 8]))
    E = min(max(8, G * int(r.choice([2, 4, 8, 16, 32]))), 256)     # E % G == 0 and E % 8 == 0
    rb = int(r.integers(0, 4))
    alpha, beta, nsat = int(r.integers(1, 9000)), int(r.integers(0, 12000)), int(r.integers(0, 300))
    rt, cfg = _rt(G, E, replica_budget=rb, alpha_ps=alpha, beta_ps=beta, n_sat=nsat, bw_bytes_per_us=770_000)
    pop = (np.arange(1, E + 1) ** -1.2)[r.permutation(E)]
    nhat = r.poisson(4000 * pop / pop.sum() * E / G, size=(G, E)).astype(np.int32)
    wbytes = 6 * 256 * 256
    windows = r.integers(0, 4 * wbytes * 1000 // 770_000 + 2, size=G).astype(np.int64)
    reps = torch.empty(G, 3, dtype=torch.int32, device="cuda")
    quota = torch.empty(G, E, G, dtype=torch.int32, device="cuda")
    stats = torch.empty(8, dtype=torch.int64, device="cuda")
    rt.plan(1, torch.from_numpy(windows).cuda(), pred_counts=torch.from_numpy(nhat).cuda(), replicas=reps,
            quota=quota, stats=stats)
    torch.cuda.synchronize()
    pc = O.PlannerConfig(G=G, E=E, replica_budget=rb, kmax=16, alpha_ps=alpha, beta_ps=beta, n_sat=nsat,
                         bw_bytes_per_us=770_000, expert_bytes=wbytes)
    plan = O.plan_greedy(nhat, windows.tolist(), pc)
    exp = np.full((G, 3), -1)
    for g in range(G):
        exp[g, :len(plan.replicas[g])] = plan.replicas[g]
    assert np.array_equal(reps.cpu().numpy(), exp)
    assert np.array_equal(quota.cpu().numpy(), plan.quota)
    st = stats.cpu().numpy()
    assert (st[0], st[1], st[2], st[3]) == (plan.iterations, len(plan.transfers), plan.maxL_before, plan.maxL_after)
    rt.close()


@pytest.mark.parametrize("budget", [3, 2])
def test_history_hook_feeds_planner(budget):
    """NEXT-3: the statistics-based one-shot policy (history of actual counts → the same
    planner); budget 2 = the paper's EPLB configuration, 2 redundant slots per rank."""
    import probe_inputs as pi
    sh = pi.C0.with_(name="hist", E=16, k=2, H=256, F=256, T=128, G=4)
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    cfg = ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h, replica_budget=budget)
    rt = ProbeRuntime(cfg)
    W = pi.router_weight(sh, 0, device="cuda")
    w13, w2 = pi.expert_weights(sh, 0, device="cuda")
    out = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    hist = torch.zeros(sh.G, sh.E, dtype=torch.int32, device="cuda")
    counts = torch.empty(sh.G, sh.E, dtype=torch.int32, device="cuda")
    total = np.zeros((sh.G, sh.E), dtype=np.int64)
    for L in range(3):
        li = pi.layer_inputs(sh, L, 0, 1.3, device="cuda")      # parity-0 router for every layer
        rt.forward(2 * L, li.x, W, None, w13, w2, out)
        rt.history_update(2 * L, hist, reset=(L == 0))
        rt.debug_layout(counts=counts)
        torch.cuda.synchronize()
        total += counts.cpu().numpy()
    assert np.array_equal(hist.cpu().numpy(), total)
    reps = torch.empty(sh.G, 3, dtype=torch.int32, device="cuda")
    win = torch.full((sh.G,), 10 ** 9, dtype=torch.int64, device="cuda")
    rt.plan(7, win, pred_counts=hist, replicas=reps)
    torch.cuda.synchronize()
    pc = O.PlannerConfig(G=sh.G, E=sh.E, replica_budget=budget, alpha_ps=1, beta_ps=0, expert_bytes=6 * sh.H * sh.F)
    plan = O.plan_greedy(total, [10 ** 9] * sh.G, pc)
    assert max(len(r) for r in plan.replicas) <= budget
    exp = np.full((sh.G, 3), -1)
    for g in range(sh.G):
        exp[g, :len(plan.replicas[g])] = plan.replicas[g]
    assert np.array_equal(reps.cpu().numpy(), exp)
    rt.close()


def test_measured_window_feeds_planner():
    """R26: probe_window returns the last measured expert-GEMM window of every rank (+ attention),
    device to device; before any forward it returns the fallback; the planner's caps then follow
    the MEASURED windows (plan bit-exact vs the oracle on the same windows)."""
    import probe_inputs as pi
    sh = pi.C0.with_(name="win", E=16, k=2, H=512, F=512, T=512, G=4)
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    wbytes = 6 * sh.H * sh.F
    bw = 770_000
    cfg = ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h, bw_bytes_per_us=bw)
    rt = ProbeRuntime(cfg)
    win = torch.empty(sh.G, dtype=torch.int64, device="cuda")
    rt.window(win, attention_ns=5, fallback_ns=1234)          # aux stream (NULL stream argument)
    torch.cuda.synchronize()
    assert win.cpu().tolist() == [1239] * sh.G                  # nothing measured yet → fallback
    li = pi.layer_inputs(sh, 0, 0, 1.5, device="cuda")
    W = pi.router_weight(sh, 0, device="cuda")
    w13, w2 = pi.expert_weights(sh, 0, device="cuda")
    out = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    rt.forward(0, li.x, W, None, w13, w2, out)
    torch.cuda.synchronize()                                     # the aux stream does not order after stream 0
    attn = 3 * wbytes * 1000 // bw // 2                          # ≈ 1.5 replicas' worth of transfer time
    rt.window(win, attention_ns=attn, fallback_ns=10 ** 12)
    torch.cuda.synchronize()
    w = win.cpu().numpy()
    assert (w > attn).all() and (w < attn + 10 ** 9).all()      # measured (not the fallback)
    # one process hosts all ranks: one grouped GEMM; rank r's window = its share by the planner's
    # compute cost Σ_active slots max(rows, n_sat) (n_sat = 0 here: the row share)
    rows = torch.empty(sh.G, sh.E // sh.G + 3, dtype=torch.int32, device="cuda")
    rt.debug_layout(group_rows=rows)
    torch.cuda.synchronize()
    share = rows.sum(dim=1).double().cpu().numpy()
    m = (w - attn).astype(np.float64)
    assert np.allclose(m / m.sum(), share / share.sum(), rtol=1e-3, atol=1e-4)   # integer ns division
    nhat = np.zeros((sh.G, sh.E), dtype=np.int32)
    nhat[:, :4] = 400                                            # rank 0's experts hot everywhere
    nhat[:, 4:] = 10
    reps = torch.empty(sh.G, 3, dtype=torch.int32, device="cuda")
    rt.plan(1, win, pred_counts=torch.from_numpy(nhat).cuda(), replicas=reps)
    torch.cuda.synchronize()
    pc = O.PlannerConfig(G=sh.G, E=sh.E, alpha_ps=1, beta_ps=0, bw_bytes_per_us=bw, expert_bytes=wbytes)
    plan = O.plan_greedy(nhat, w.tolist(), pc)
    assert plan.caps == O.replica_caps(w.tolist(), pc)
    exp = np.full((sh.G, 3), -1)
    for g in range(sh.G):
        exp[g, :len(plan.replicas[g])] = plan.replicas[g]
    assert np.array_equal(reps.cpu().numpy(), exp)
    rt.close()

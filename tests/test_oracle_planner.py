"""Pins for the oracle's planner (a4, Algorithm 1) and materialization (a5).

Pinned by: the SPEC worked example (S:313/325/334), a hand-derived 4-rank trace
with a communication term (tests/golden/planner_examples.json), trivial cases
(S:323-324), window-boundary rules, the Eq. 7 brute-force optimum
(placement enumeration × exact MILP over integer splits) as a bound on every
tiny instance and equality on compute-only instances, and the invariants S:337-342.
"""
import itertools

import numpy as np
import pytest

from oracle import (PlannerConfig, imbalance_ratio, materialize, plan_greedy, rank_costs,
                    replica_caps, static_plan, token_loads)

BIG = 10 ** 12


def cfg_from(d, **kw):
    base = dict(G=d["G"], E=d["E"], replica_budget=d["replica_budget"], kmax=d["kmax"],
                alpha_ps=d["alpha_ps"], beta_ps=d["beta_ps"], n_sat=d["n_sat"],
                bw_bytes_per_us=10 ** 6, expert_bytes=1)
    base.update(kw)
    return PlannerConfig(**base)


@pytest.mark.parametrize("name", ["spec_worked_example", "hand_trace_g4_comm"])
def test_planner_golden(golden, name):
    d = golden["planner_examples"][name]
    cfg = cfg_from(d)
    p = plan_greedy(np.array(d["nhat"]), [BIG] * cfg.G, cfg)
    ex = d["expect"]
    assert p.replicas == ex["replicas"]
    assert p.L_before == ex["L_before"]
    assert p.L_after == ex["L_after"]
    assert p.iterations == ex["iterations"]
    assert [list(t) for t in p.transfers] == ex["transfers"]
    if "quota" in ex:
        assert p.quota.tolist() == ex["quota"]
        assert token_loads(p.quota) == ex["loads_after"]
        assert imbalance_ratio(token_loads(p.quota)) == ex["ir_after"]


def test_uniform_gives_empty_plan():
    cfg = PlannerConfig(G=4, E=8, alpha_ps=3, beta_ps=2, n_sat=4)
    nhat = np.full((4, 8), 10)
    p = plan_greedy(nhat, [BIG] * 4, cfg)
    assert p.iterations == 0 and all(r == [] for r in p.replicas)
    assert np.array_equal(p.quota, static_plan(nhat, cfg))


@pytest.mark.parametrize("kw", [dict(replica_budget=0), dict(windows=0)])
def test_zero_budget_or_window_gives_baseline(kw):
    cfg = PlannerConfig(G=2, E=2, replica_budget=kw.get("replica_budget", 3))
    nhat = np.array([[150, 50], [150, 50]])
    w = [kw.get("windows", BIG)] * 2
    p = plan_greedy(nhat, w, cfg)
    assert p.iterations == 0 and p.replicas == [[], []]
    assert np.array_equal(p.quota, static_plan(nhat, cfg))


def test_window_boundary_inclusive_and_caps():
    # Eq. 6: n·𝒲/BW ≤ window.  𝒲 = 1000 B, BW = 1000 B/µs → 1 µs per expert.
    cfg = PlannerConfig(G=2, E=2, bw_bytes_per_us=1000, expert_bytes=1000)
    assert replica_caps([1000, 999, 2000, 10 ** 9], cfg) == [1, 0, 2, 3]
    nhat = np.array([[150, 50], [150, 50]])
    assert plan_greedy(nhat, [1000, 1000], cfg).replicas == [[], [0]]   # exactly equal → allowed
    assert plan_greedy(nhat, [1000, 999], cfg).replicas == [[], []]     # receiver short by 1 ns
    assert plan_greedy(nhat, [999, 1000], cfg).replicas == [[], []]     # sender side (dual check)


def test_receiver_at_budget_rejected():
    # rank 1 would take 4 replicas of rank 0's hot experts; budget 3 stops it
    cfg = PlannerConfig(G=2, E=8, replica_budget=3)
    nhat = np.array([[0, 0, 0, 0, 0, 0, 0, 0], [100, 90, 80, 70, 1, 1, 1, 1]])
    p = plan_greedy(nhat, [BIG, BIG], cfg)
    assert len(p.replicas[1]) <= 3
    assert p.replicas[1] == sorted(p.replicas[1])


def _check_invariants(nhat, p, cfg):
    G, E = cfg.G, cfg.E
    q = p.quota
    assert np.array_equal(q.sum(axis=2), nhat)                                   # conservation
    for s in range(G):
        for e in range(E):
            for t in range(G):
                if q[s, e, t] > 0:
                    assert e // cfg.EL == t or e in p.replicas[t]                # validity
    for r in range(G):
        assert len(p.replicas[r]) <= p.caps[r]                                   # caps (Δin)
        assert sum(1 for (_, src, _) in p.transfers if src == r) <= p.caps[r]    # caps (Δout)
    assert p.maxL_after <= p.maxL_before                                         # monotone
    assert p.iterations <= cfg.kmax                                              # termination
    for (e, src, dst) in p.transfers:                                            # locality pinning
        assert q[src, e, src] == nhat[src, e]
        assert src == e // cfg.EL
    hosts = [set(range(r * cfg.EL, (r + 1) * cfg.EL)) | set(p.replicas[r]) for r in range(G)]
    assert rank_costs(q, hosts, cfg) == p.L_after                                # L consistent


@pytest.mark.parametrize("seed", range(40))
def test_planner_invariants_random(seed):
    r = np.random.default_rng(seed)
    G = int(r.choice([2, 4, 8]))
    E = G * int(r.choice([1, 2, 4, 8]))
    cfg = PlannerConfig(G=G, E=E, replica_budget=int(r.integers(0, 4)), kmax=16,
                        alpha_ps=int(r.integers(1, 10)), beta_ps=int(r.integers(0, 10)),
                        n_sat=int(r.integers(0, 50)), bw_bytes_per_us=1000, expert_bytes=1000)
    pop = r.pareto(1.0, E) + 0.01
    nhat = r.poisson(200 * pop / pop.sum() * E, size=(G, E))
    windows = r.integers(0, 4000, size=G)
    p = plan_greedy(nhat, windows, cfg)
    _check_invariants(nhat, p, cfg)
    p2 = plan_greedy(nhat, windows, cfg)                                         # determinism
    assert np.array_equal(p.quota, p2.quota) and p.replicas == p2.replicas


# ---------------------------------------------------------------------------
# Brute-force optimum of Eq. 7 on tiny instances
# ---------------------------------------------------------------------------

def eq7_optimum(nhat, cfg, caps):
    """min over placements (|Δin_r| ≤ cap_r, senders = home with #out ≤ cap) of the exact
    MILP min_{split} max_r L_r, L_r = α Σ c(m_er) + β max(in_r, out_r), integer split,
    c(m) = max(m, n_sat)·[m > 0].  No locality pinning (Eq. 7 has none)."""
    from scipy.optimize import LinearConstraint, milp, Bounds
    G, E, EL = cfg.G, cfg.E, cfg.EL
    per_rank = []
    for r in range(G):
        others = [e for e in range(E) if e // EL != r]
        opts = []
        for kk in range(0, caps[r] + 1):
            opts.extend(itertools.combinations(others, kk))
        per_rank.append(opts)
    best = None
    for placement in itertools.product(*per_rank):
        n_out = [0] * G
        for r in range(G):
            for e in placement[r]:
                n_out[e // EL] += 1
        if any(n_out[r] > caps[r] for r in range(G)):
            continue
        hosts = [set(range(r * EL, (r + 1) * EL)) | set(placement[r]) for r in range(G)]
        # variables: x[s,e,t] for t hosting e; c[e,t], y[e,t] for hosted; u_r (comm); z
        var = {}
        def v(key):
            if key not in var:
                var[key] = len(var)
            return var[key]
        for s in range(G):
            for e in range(E):
                for t in range(G):
                    if e in hosts[t]:
                        v(("x", s, e, t))
        for t in range(G):
            for e in sorted(hosts[t]):
                v(("c", e, t)); v(("y", e, t))
            v(("u", t))
        z = v(("z",))
        nv = len(var)
        A, lo, hi = [], [], []
        def row(coefs, l, h):
            a = np.zeros(nv)
            for k_, c_ in coefs:
                a[k_] += c_
            A.append(a); lo.append(l); hi.append(h)
        M = int(nhat.sum()) + 1
        for s in range(G):
            for e in range(E):
                row([(var[("x", s, e, t)], 1) for t in range(G) if e in hosts[t]], nhat[s, e], nhat[s, e])
        for t in range(G):
            for e in sorted(hosts[t]):
                m = [(var[("x", s, e, t)], 1) for s in range(G)]
                row(m + [(var[("y", e, t)], -M)], -np.inf, 0)                    # m ≤ M y
                row([(var[("c", e, t)], 1)] + [(k_, -1) for k_, _ in m], 0, np.inf)   # c ≥ m
                row([(var[("c", e, t)], 1), (var[("y", e, t)], -cfg.n_sat)], 0, np.inf)  # c ≥ n_sat y
            inn = [(var[("x", s, e, t)], 1) for s in range(G) if s != t for e in range(E) if e in hosts[t]]
            out = [(var[("x", t, e, tt)], 1) for tt in range(G) if tt != t for e in range(E) if e in hosts[tt]]
            row([(var[("u", t)], 1)] + [(k_, -1) for k_, _ in inn], 0, np.inf)
            row([(var[("u", t)], 1)] + [(k_, -1) for k_, _ in out], 0, np.inf)
            row([(z, 1)] + [(var[("c", e, t)], -cfg.alpha_ps) for e in sorted(hosts[t])]
                + [(var[("u", t)], -cfg.beta_ps)], 0, np.inf)
        cost = np.zeros(nv); cost[z] = 1
        integrality = np.ones(nv)
        ub = np.full(nv, np.inf)
        for key, i in var.items():
            if key[0] == "y":
                ub[i] = 1
        res = milp(cost, constraints=LinearConstraint(np.array(A), lo, hi),
                   integrality=integrality, bounds=Bounds(np.zeros(nv), ub))
        assert res.status == 0
        val = int(round(res.fun))
        if best is None or val < best:
            best = val
    return best


@pytest.mark.parametrize("seed", range(6))
def test_greedy_equals_eq7_optimum_compute_only(seed):
    """compute-only cost (β=0, n_sat=0), Rb=3, G=2, E=8, T=64, k=2:
    the greedy reaches the Eq. 7 optimum."""
    r = np.random.default_rng(1000 + seed)
    G, E, T, k = 2, 8, 64, 2
    pop = np.arange(1, E + 1, dtype=float) ** -1.2
    pop = pop[r.permutation(E)]
    nhat = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        for t in range(T):
            keys = np.log(pop) + r.gumbel(size=E)
            for e in np.argsort(-keys)[:k]:
                nhat[s, e] += 1
    cfg = PlannerConfig(G=G, E=E, replica_budget=3, alpha_ps=1, beta_ps=0, n_sat=0)
    p = plan_greedy(nhat, [BIG] * G, cfg)
    opt = eq7_optimum(nhat, cfg, p.caps)
    assert p.maxL_after >= opt
    assert p.maxL_after == opt


@pytest.mark.parametrize("seed", range(4))
def test_greedy_bounded_below_by_eq7_with_comm(seed):
    """With a comm term the greedy is a heuristic (App. A.2): greedy ≥ opt always; report only."""
    r = np.random.default_rng(2000 + seed)
    G, E = 2, 4
    nhat = r.integers(0, 40, size=(G, E))
    nhat[0, 0] += 60
    cfg = PlannerConfig(G=G, E=E, replica_budget=2, alpha_ps=4, beta_ps=2, n_sat=3)
    p = plan_greedy(nhat, [BIG] * G, cfg)
    opt = eq7_optimum(nhat, cfg, p.caps)
    assert p.maxL_after >= opt
    assert p.maxL_after <= p.maxL_before


# ---------------------------------------------------------------------------
# a5 materialize (R23)
# ---------------------------------------------------------------------------

def test_materialize_static_and_conservation():
    G, E = 4, 8
    r = np.random.default_rng(5)
    n = r.integers(0, 30, size=(G, E))
    split = materialize(n, None, [[] for _ in range(G)], G, E)
    for s in range(G):
        for e in range(E):
            assert split[s, e, e // 2] == n[s, e] and split[s, e].sum() == n[s, e]


def test_materialize_proportional_and_leftover():
    G, E = 3, 3
    quota = np.zeros((G, E, G), dtype=np.int64)
    quota[0, 0] = [4, 4, 2]           # P=10; n=7: floors 2.8→2, 2.8→2, 1.4→1 → leftover 2 to t=0 (tie → lowest)
    quota[1, 0] = [0, 0, 0]           # P=0: s=1 does not host e0 → home 0
    quota[2, 0] = [1, 0, 3]           # s=2 hosts replica of e0: P=4, n=5: 1, 0, 3 (5*3//4=3) → left 1 → t=2
    n = np.zeros((G, E), dtype=np.int64)
    n[0, 0], n[1, 0], n[2, 0] = 7, 6, 5
    reps = [[], [0], [0]]
    split = materialize(n, quota, reps, G, E)
    assert split[0, 0].tolist() == [4, 2, 1]
    assert split[1, 0].tolist() == [0, 6, 0]          # P=0 and s=1 hosts a replica → stays on s
    assert split[2, 0].tolist() == [1, 0, 4]
    reps = [[], [], [0]]
    split = materialize(n, quota, reps, G, E)
    assert split[1, 0].tolist() == [6, 0, 0]          # not hosted on s → home(e)

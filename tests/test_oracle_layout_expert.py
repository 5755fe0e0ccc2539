"""Pins for the oracle's dispatch layout (a6), expert FFN (a7), combine (a8) and
the analytical model (Eq. 1, 2, 4, 6; slot banks).

Layout is pinned against an independent sort-based construction of R24's order;
the expert FFN against torch's dense SwiGLU (G=1, E=1, k=1 reduces to a dense MLP);
combine against the identity-expert conservation law; cost model against SPEC.
"""
import numpy as np
import pytest
import torch

import probe_inputs as pi
from oracle import (PlannerConfig, combine, dispatch_layout, exposed_overhead, expert_compute_time,
                    imbalance_ratio, layer_reference, materialize, moe_layer_outputs, plan_greedy,
                    replica_slot_schedule, swiglu_expert, traffic_volumes, transfer_latency)


def _random_ids(r, G, T, E, k):
    ids = []
    for s in range(G):
        ids.append(np.stack([r.choice(E, size=k, replace=False) for _ in range(T)]))
    return ids


@pytest.mark.parametrize("seed", range(5))
def test_layout_matches_sort_construction(seed):
    r = np.random.default_rng(seed)
    G, E, T, k = 4, 8, 37, 3
    ids = _random_ids(r, G, T, E, k)
    n = np.stack([np.bincount(i.reshape(-1), minlength=E) for i in ids])
    cfg = PlannerConfig(G=G, E=E, alpha_ps=1, beta_ps=1)
    plan = plan_greedy(n + r.integers(0, 3, size=n.shape), [10 ** 9] * G, cfg)   # plan on noisy n̂
    split = materialize(n, plan.quota, plan.replicas, G, E)
    lay = dispatch_layout(ids, split, plan.replicas, G, E)
    # independent construction: list every (token, slot) with its destination; sort by
    # (dest, local slot, src, token) and number rows per destination.
    recs = []
    for s in range(G):
        for t in range(T):
            for j in range(k):
                d = int(lay.dest[s][t, j])
                e = int(ids[s][t, j])
                slots = list(range(d * (E // G), (d + 1) * (E // G))) + sorted(plan.replicas[d])
                recs.append((d, slots.index(e), s, t, j))
    recs.sort()
    counters = [0] * G
    for (d, ls, s, t, j) in recs:
        assert lay.row[s][t, j] == counters[d]
        counters[d] += 1
    assert counters == [len(x) for x in lay.rows]
    # each (s,e,t) destination count equals the split (dispatch follows the materialized plan)
    for s in range(G):
        for e in range(E):
            for d in range(G):
                assert int(((ids[s] == e) & (lay.dest[s] == d)).sum()) == split[s, e, d]
    # tokens of (s,e) fill destinations in ascending order along ascending token index
    for s in range(G):
        for e in range(E):
            dd = lay.dest[s][ids[s] == e]
            assert np.all(np.diff(dd) >= 0)


def test_layout_static_ep_identity():
    r = np.random.default_rng(3)
    G, E, T, k = 2, 8, 20, 2
    ids = _random_ids(r, G, T, E, k)
    n = np.stack([np.bincount(i.reshape(-1), minlength=E) for i in ids])
    lay = dispatch_layout(ids, materialize(n, None, [[], []], G, E), [[], []], G, E)
    for s in range(G):
        assert np.array_equal(lay.dest[s], ids[s] // (E // G))     # every token to its expert's home
    assert [sum(gz) for gz in lay.group_sizes] == [int(n[:, :4].sum()), int(n[:, 4:].sum())]


def test_swiglu_dense_reduction_vs_torch():
    r = np.random.default_rng(0)
    T, H, F = 9, 16, 24
    x = r.standard_normal((T, H))
    W13 = r.standard_normal((2 * F, H))
    W2 = r.standard_normal((H, F))
    y = swiglu_expert(x, W13, W2)
    xt = torch.from_numpy(x)
    ref = (torch.nn.functional.silu(xt @ torch.from_numpy(W13[:F]).T) * (xt @ torch.from_numpy(W13[F:]).T)) \
        @ torch.from_numpy(W2).T
    assert np.allclose(y, ref.numpy(), rtol=1e-13, atol=1e-13)
    # G=1, E=1, k=1: the MoE layer is the dense MLP (g = 1)
    out = moe_layer_outputs(x, np.zeros((T, 1), dtype=np.int64), np.ones((T, 1)), {0: W13}, {0: W2})
    assert np.allclose(out, ref.numpy(), rtol=1e-13, atol=1e-13)


def test_combine_identity_expert_conservation():
    r = np.random.default_rng(1)
    T, k, H = 11, 4, 8
    x = r.standard_normal((T, H))
    g = r.random((T, k))
    g /= g.sum(axis=1, keepdims=True)
    y = np.repeat(x[:, None, :], k, axis=1)        # identity expert: y := x
    assert np.allclose(combine(g, y), x, atol=1e-15)


def test_layer_output_independent_of_plan():
    shape = pi.C0
    li = pi.layer_inputs(shape, step=0, layer=0, zipf_s=1.5)
    W = pi.bf16_to_numpy_f64(pi.router_weight(shape, 0))
    w13, w2 = pi.expert_weights(shape, 0)
    W13 = {e: pi.bf16_to_numpy_f64(w13[e]) for e in range(shape.E)}
    W2 = {e: pi.bf16_to_numpy_f64(w2[e]) for e in range(shape.E)}
    xs = [pi.bf16_to_numpy_f64(li.x[r]) for r in range(shape.G)]
    a = layer_reference(xs, W, None, shape.k, None, shape.G, shape.E, W13, W2)
    cfg = PlannerConfig(G=shape.G, E=shape.E, alpha_ps=1, beta_ps=0)
    plan = plan_greedy(a["n"], [10 ** 9] * shape.G, cfg)
    b = layer_reference(xs, W, None, shape.k, plan, shape.G, shape.E, W13, W2)
    assert any(plan.replicas)
    for s in range(shape.G):
        assert np.array_equal(a["out"][s], b["out"][s])             # A19 semantic equivalence
    assert imbalance_ratio(b["split"].sum(axis=(0, 1))) <= imbalance_ratio(a["split"].sum(axis=(0, 1)))


def test_costmodel_spec_pins(golden):
    sp = golden["spec_pins"]
    for c in sp["ir"]["cases"]:
        assert imbalance_ratio(c["loads"]) == pytest.approx(c["ir"], rel=1e-15)
    for c in sp["eq2"]["cases"]:
        assert expert_compute_time(c["n"], c["Fbar"], c["Fpeak"], c["n_sat"]) == pytest.approx(c["t"], rel=1e-12)
    e4 = sp["eq4"]
    split = np.zeros((2, 2, 2), dtype=np.int64)
    split[0, 1, 1] = e4["tokens"]                     # 100 tokens r0 → expert hosted on r1
    vin, vout = traffic_volumes(split, e4["H_bytes"])
    assert vout[0] == e4["vin_lambda1"] and vin[1] == e4["vin_lambda1"]
    vin, _ = traffic_volumes(split, e4["H_bytes"], lam_in=[1, 2])
    assert vin[1] == e4["vin_lambda2"]
    for c in sp["eq6"]["cases"]:
        assert transfer_latency(c["n_in"], c["n_out"], c["W"], c["bw"]) == pytest.approx(c["t"], rel=1e-12)
    assert exposed_overhead([5e-4, 1e-4], [3e-4, 2e-4]) == pytest.approx(2e-4)
    assert exposed_overhead([1e-4], [2e-4]) == 0.0
    s = replica_slot_schedule([[[7, 8, 9]], [[1, 2, 3]]])
    assert s == sp["slots"]["alternating"]
    with pytest.raises(ValueError):
        replica_slot_schedule([[[1, 2, 3, 4]]])


def test_integer_cost_is_eq2():
    # c(m) = max(m, n_sat) (m>0) is Eq. 2 in units of F̄/F_peak
    from oracle.probe_oracle import _c
    for m in [0, 1, 63, 64, 256, 1000]:
        assert _c(m, 256) * 1e9 / 1e15 == pytest.approx(expert_compute_time(m, 1e9, 1e15, 256))


def test_moe_outputs_ranks_matches_per_token_brute_force():
    """The expert-outer loop (moe_outputs_ranks) against a per-(token, slot) brute force
    written from the definition out_t = Σ_j g_tj · SwiGLU_{ids_tj}(x_t), on sampled tokens."""
    from oracle import moe_outputs_ranks
    r = np.random.default_rng(5)
    G, T, H, F, E, k = 3, 13, 8, 12, 5, 2
    W13 = {e: r.standard_normal((2 * F, H)) for e in range(E)}
    W2 = {e: r.standard_normal((H, F)) for e in range(E)}
    xs = [r.standard_normal((T, H)) for _ in range(G)]
    ids = [np.stack([r.choice(E, size=k, replace=False) for _ in range(T)]) for _ in range(G)]
    gs = [r.random((T, k)) for _ in range(G)]
    toks = [[0, 4, 12], list(range(T)), [7]]
    outs = moe_outputs_ranks(xs, ids, gs, W13, W2, toks)
    for s in range(G):
        for i, t in enumerate(toks[s]):
            want = np.zeros(H)
            for j in range(k):
                e = ids[s][t, j]
                gg = W13[e][:F] @ xs[s][t]
                uu = W13[e][F:] @ xs[s][t]
                want += gs[s][t, j] * (W2[e] @ (gg / (1 + np.exp(-gg)) * uu))
            assert np.allclose(outs[s][i], want, rtol=1e-12, atol=1e-12)
        assert np.allclose(outs[s], moe_layer_outputs(xs[s], ids[s], gs[s], W13, W2, toks[s]), rtol=1e-13, atol=1e-13)

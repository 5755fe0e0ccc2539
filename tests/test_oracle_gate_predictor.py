"""Pins for the oracle's gate (a1) and lookahead predictor (a2).

Each pin is fixed by something other than the oracle itself: SPEC worked
examples, the Hadamard-encoded design (closed-form logits v_j/16), closed forms
(softmax over the selected logits, Ŵ2 = 0 ⇒ prior, x = 0 ⇒ bias), an
independent library rounding routine (torch bf16), and hand-computed values.
"""
import math

import numpy as np
import pytest
import torch

import probe_inputs as pi
from oracle import (gate, predictor_logits, predict_counts, round_bf16, router_logits, silu,
                    topk_ids)


def test_topk_spec_examples(golden):
    for c in golden["spec_pins"]["topk"]["cases"]:
        ids = topk_ids(np.array([c["logits"]], dtype=float), c["k"])
        assert sorted(ids[0].tolist()) == c["set"]


def test_topk_slot_order_and_shift_invariance():
    l = np.array([[0.5, 2.0, 2.0, -1.0, 3.0]])
    assert topk_ids(l, 3)[0].tolist() == [4, 1, 2]       # logit ↓ then id ↑ (R3/R4)
    assert topk_ids(l + 7.25, 3)[0].tolist() == [4, 1, 2]  # S:412 shift invariance


def expected_gate_from_design(d: pi.RankDesign, k: int):
    """Expected routing derived from the DESIGN (not from logits): candidates are the
    designed slots plus the boundary-tie expert with their numerators; order by
    (numerator ↓, id ↑) — the paper's tie rule R3/R4 applied to the designed values."""
    T = d.S.shape[0]
    out = np.zeros((T, k), dtype=np.int64)
    for t in range(T):
        cand = [(int(d.numer[t, j]), int(d.S[t, j])) for j in range(k)]
        if d.tie_e[t] >= 0:
            cand.append((int(d.numer[t, k - 1]), int(d.tie_e[t])))
        cand.sort(key=lambda p: (-p[0], p[1]))
        out[t] = [e for _, e in cand[:k]]
    return out


@pytest.mark.parametrize("shape", [pi.C0, pi.C0.with_(E=16, k=4, H=512, T=96)])
def test_gate_reproduces_hadamard_design(shape):
    li = pi.layer_inputs(shape, step=3, layer=0, zipf_s=1.2)
    W = pi.bf16_to_numpy_f64(pi.router_weight(shape, 0))
    n_ties = 0
    for r in range(shape.G):
        x = pi.bf16_to_numpy_f64(li.x[r])
        d = li.designs[r]
        l = router_logits(x, W, None)
        # closed form: logit = v/16 on the designed experts, 0 elsewhere (Hadamard orthogonality)
        exp_l = np.zeros_like(l)
        for t in range(shape.T):
            for j in range(shape.k):
                exp_l[t, d.S[t, j]] = d.numer[t, j] / 16.0
            if d.tie_e[t] >= 0:
                exp_l[t, d.tie_e[t]] = d.numer[t, shape.k - 1] / 16.0
        assert np.array_equal(l, exp_l)
        ids, g, counts = gate(x, W, None, shape.k)
        assert np.array_equal(ids, expected_gate_from_design(d, shape.k))
        n_ties += int((d.tie_e >= 0).sum())
        # softmax over the selected logits: closed form and Σ g = 1
        sel = np.take_along_axis(exp_l, ids, axis=1)
        ref = np.exp(sel) / np.exp(sel).sum(axis=1, keepdims=True)
        assert np.allclose(g, ref, rtol=0, atol=1e-15)
        assert np.allclose(g.sum(axis=1), 1.0, atol=1e-15)
        assert counts.sum() == shape.T * shape.k
        exp_ids = expected_gate_from_design(d, shape.k)
        assert np.array_equal(counts, np.bincount(exp_ids.reshape(-1), minlength=shape.E))


def test_gate_bias_shifts_selection():
    x = np.eye(3)
    W = np.eye(3)
    b = np.array([0.0, 0.0, 2.0])
    ids, g, _ = gate(x, W, b, 1)
    assert ids[:, 0].tolist() == [2, 2, 2]          # bias 2 beats logit 1 (P:381 b_L term)
    ids, g, _ = gate(x, W, None, 1)
    assert ids[:, 0].tolist() == [0, 1, 2]


def test_round_bf16_matches_torch():
    r = np.random.default_rng(0)
    a = np.concatenate([r.standard_normal(20000) * 10.0 ** r.integers(-6, 6, 20000),
                        [1 + 2 ** -8, 1 + 3 * 2 ** -8, -1 - 2 ** -8, 0.0, 1.0]])
    ref = torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(round_bf16(a), ref)


def test_predictor_zero_residual_is_prior():
    shape = pi.C0
    li = pi.layer_inputs(shape, step=1, layer=0)
    Wn = pi.bf16_to_numpy_f64(pi.router_weight(shape, 1))
    w1, w2 = pi.predictor_residual(shape, 1, zero=True)
    x = pi.bf16_to_numpy_f64(li.x[0])
    l, _ = predictor_logits(x, Wn, None, pi.bf16_to_numpy_f64(w1), pi.bf16_to_numpy_f64(w2))
    assert np.array_equal(l, router_logits(x, Wn, None))   # S:390, P:384 zero-init
    # prior reproduces the encoded prediction P_t exactly (design, not oracle)
    d = li.designs[0]
    for t in range(shape.T):
        assert topk_ids(l[t:t + 1], shape.k)[0].tolist() == list(d.P[t])


def test_predictor_x_zero_gives_bias():
    r = np.random.default_rng(1)
    W = r.standard_normal((5, 7))
    b = r.standard_normal(5)
    W1 = r.standard_normal((3, 7))
    W2 = r.standard_normal((5, 3))
    l, a = predictor_logits(np.zeros((2, 7)), W, b, W1, W2)
    assert np.array_equal(l, np.tile(b, (2, 1)))            # σ(0) = 0
    assert np.all(a == 0)


def test_predictor_hand_example():
    # 1 token, H=2, E=2, h=1; every value hand-computed:
    # prior = W x + b = [1*1 + 2*0.5 + 0.25, -1*1 + 0] = [2.25, -1.0]
    # z = W1 x = 1*1 + 2*0.5 = 2;  SiLU(2) = 2/(1+e^-2) = 1.7615941559557646
    # bf16(1.76159...): 8 significant bits, value in [1,2) → 7 fraction bits:
    #   1.76159 * 128 = 225.48 → 225 → 225/128 = 1.7578125
    x = np.array([[1.0, 0.5]])
    W = np.array([[1.0, 2.0], [-1.0, 0.0]])
    b = np.array([0.25, 0.0])
    W1 = np.array([[1.0, 2.0]])
    W2 = np.array([[0.5], [-2.0]])
    s2 = 2.0 / (1.0 + math.exp(-2.0))
    assert abs(s2 - 1.7615941559557646) < 1e-15
    a_bf16 = 225.0 / 128.0      # 1.76159*128 = 225.48 → nearest integer 225 (exponent 0: 7 frac bits)
    l, a = predictor_logits(x, W, b, W1, W2)
    assert a[0, 0] == a_bf16
    assert np.array_equal(l, np.array([[2.25 + 0.5 * a_bf16, -1.0 - 2.0 * a_bf16]]))
    l2, a2 = predictor_logits(x, W, b, W1, W2, round_activation=False)
    assert a2[0, 0] == s2


def test_predict_counts_bounded_residual_keeps_design():
    shape = pi.C0.with_(E=16, k=4, H=512, T=80)
    li = pi.layer_inputs(shape, step=2, layer=1)     # parity 1 → next layer parity 0
    Wn = pi.bf16_to_numpy_f64(pi.router_weight(shape, 0))
    w1, w2 = pi.predictor_residual(shape, 0)
    for r in range(shape.G):
        x = pi.bf16_to_numpy_f64(li.x[r])
        l, a = predictor_logits(x, Wn, None, pi.bf16_to_numpy_f64(w1), pi.bf16_to_numpy_f64(w2))
        res = l - router_logits(x, Wn, None)
        assert np.abs(res).max() < 2 ** -6        # bounded residual (generator contract)
        assert np.abs(res).max() > 0
        counts, ids = predict_counts(x, Wn, None, pi.bf16_to_numpy_f64(w1), pi.bf16_to_numpy_f64(w2), shape.k)
        assert np.array_equal(ids, li.designs[r].P)
        assert np.array_equal(counts, np.bincount(li.designs[r].P.reshape(-1), minlength=shape.E))


def test_designed_prediction_accuracy_near_paper():
    # P:390 "≈90% Top-K accuracy": encoded accuracy a = 0.9 → measured overlap ≈ 0.9
    shape = pi.C0.with_(E=64, k=4, H=256, T=2048, G=1)
    d = pi.design_rank(shape, 0, 0, 0, 1.0, 0.9)
    acc = np.mean([len(set(d.P[t]) & set(d.S_next[t])) / shape.k for t in range(shape.T)])
    assert 0.88 < acc < 0.92


def test_silu_values():
    assert silu(np.array([0.0]))[0] == 0.0
    assert abs(silu(np.array([1.0]))[0] - 1.0 / (1.0 + math.exp(-1.0))) < 1e-16


def test_relabel_residual_moves_predicted_sets_exactly():
    """probe_inputs.predictor_residual_relabel: Eq. (P) with this residual must predict the
    designed set P_t relabelled by the cyclic shift σ on the seeded set D, with every logit a
    multiple of 1/16 (so the GPU's fp32 logits equal the oracle's), and n̂ must differ from the
    prior-only counts (the residual matters for the plan)."""
    import probe_inputs as pi
    from oracle import predictor_logits, topk_ids
    sh = pi.C0.with_(name="rl", E=32, k=4, H=512, F=64, T=300, G=2)
    li = pi.layer_inputs(sh, 0, 0, 1.2)
    W = pi.bf16_to_numpy_f64(pi.router_weight(sh, 1))
    w1, w2 = pi.predictor_residual_relabel(sh, 1)
    W1, W2 = pi.bf16_to_numpy_f64(w1), pi.bf16_to_numpy_f64(w2)
    D = np.nonzero(W2.min(axis=1) < 0)[0]
    sig = {int(D[i]): int(np.roll(D, -1)[i]) for i in range(len(D))}
    changed = False
    for r in range(sh.G):
        x = pi.bf16_to_numpy_f64(li.x[r])
        l, a = predictor_logits(x, W, None, W1, W2)
        assert np.array_equal(l * 16, np.round(l * 16)), "logits off the 1/16 grid"
        P = li.designs[r].P
        want = np.sort(np.vectorize(lambda e: sig.get(int(e), int(e)))(P), axis=1)
        got = np.sort(topk_ids(l, sh.k), axis=1)
        assert np.array_equal(got, want)
        prior, _ = predictor_logits(x, W, None, None, None)
        changed |= not np.array_equal(np.sort(topk_ids(prior, sh.k), axis=1), got)
    assert changed

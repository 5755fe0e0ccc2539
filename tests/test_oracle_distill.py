"""Pins for the distillation oracle (oracle/distill_oracle.py, R33-R37).

Each pin is independent of the oracle's own arithmetic: central finite differences of the
loss, torch.autograd in fp64 as a second backprop, Gibbs' inequality and its equality
case, closed forms at a zero residual, the zero column sums of the softmax Jacobian,
monotone full-batch descent, and SPEC's fidelity examples plus brute force.
"""
import numpy as np
import pytest
import torch

import oracle as O


def _problem(seed=0, N=24, H=16, h=8, E=8, scale=0.4, drift=0.3):
    r = np.random.default_rng(seed)
    x = r.normal(size=(N, H))
    xn = x + drift * r.normal(size=(N, H))
    W = r.normal(size=(E, H)) * scale
    b = r.normal(size=E) * 0.1
    W1 = r.normal(size=(h, H)) * scale
    W2 = r.normal(size=(E, h)) * scale
    return x, xn, W, b, W1, W2


def test_gradients_match_central_finite_differences():
    x, xn, W, b, W1, W2 = _problem(1)
    _, g1, g2, _ = O.distill_grads(x, xn, W, b, W1, W2, round_activation=False)
    r = np.random.default_rng(5)
    eps = 1e-6
    for M, G, which in ((W1, g1, 1), (W2, g2, 2)):
        for _ in range(12):
            i, j = r.integers(M.shape[0]), r.integers(M.shape[1])
            Mp, Mm = M.copy(), M.copy()
            Mp[i, j] += eps
            Mm[i, j] -= eps
            args_p = (Mp, W2) if which == 1 else (W1, Mp)
            args_m = (Mm, W2) if which == 1 else (W1, Mm)
            fd = (O.distill_loss(x, xn, W, b, *args_p, round_activation=False)
                  - O.distill_loss(x, xn, W, b, *args_m, round_activation=False)) / (2 * eps)
            assert abs(fd - G[i, j]) <= 1e-6 * max(1.0, abs(G[i, j])), (which, i, j, fd, G[i, j])


def test_gradients_match_torch_autograd():
    x, xn, W, b, W1, W2 = _problem(2, N=40, H=32, h=16, E=16)
    loss, g1, g2, _ = O.distill_grads(x, xn, W, b, W1, W2, round_activation=False)
    tx, txn, tW, tb = (torch.tensor(v, dtype=torch.float64) for v in (x, xn, W, b))
    t1 = torch.tensor(W1, dtype=torch.float64, requires_grad=True)
    t2 = torch.tensor(W2, dtype=torch.float64, requires_grad=True)
    lhat = tx @ tW.T + tb + torch.nn.functional.silu(tx @ t1.T) @ t2.T
    p = torch.softmax(txn @ tW.T + tb, dim=1)
    tl = -(p * torch.log_softmax(lhat, dim=1)).sum()
    tl.backward()
    assert abs(tl.item() - loss) <= 1e-10 * abs(loss)
    assert np.allclose(t1.grad.numpy(), g1, rtol=1e-10, atol=1e-12)
    assert np.allclose(t2.grad.numpy(), g2, rtol=1e-10, atol=1e-12)


def test_gibbs_inequality_and_equality_case():
    x, xn, W, b, W1, W2 = _problem(3)
    f = O.distill_forward(x, xn, W, b, W1, W2)
    p = O.softmax(f["t"])
    entropy = float(-(p * np.log(p)).sum())
    assert O.distill_loss(x, xn, W, b, W1, W2) >= entropy
    # no drift and a zero residual: student == teacher, loss == H(p), every gradient 0
    loss, g1, g2, _ = O.distill_grads(x, x, W, b, W1, np.zeros_like(W2))
    f0 = O.softmax(x @ W.T + b)
    assert abs(loss - float(-(f0 * np.log(f0)).sum())) < 1e-9
    assert np.abs(g1).max() < 1e-12 and np.abs(g2).max() < 1e-12


def test_zero_residual_closed_forms():
    x, xn, W, b, W1, W2 = _problem(4)
    loss, g1, g2, f = O.distill_grads(x, xn, W, b, W1, np.zeros_like(W2))
    assert np.array_equal(g1, np.zeros_like(g1))            # Ŵ² = 0 blocks the path to Ŵ¹
    q = O.softmax(x @ W.T + b)                               # student == frozen prior
    p = O.softmax(xn @ W.T + b)
    a = O.round_bf16(O.silu(x @ W1.T))
    assert np.allclose(g2, (q - p).T @ a, rtol=1e-12, atol=1e-14)


def test_softmax_jacobian_columns_sum_to_zero():
    x, xn, W, b, W1, W2 = _problem(6)
    _, _, g2, f = O.distill_grads(x, xn, W, b, W1, W2)
    # Σ_e (q − p)_te = 0 for every token ⇒ Σ_e ∇Ŵ²[e, j] = 0 for every j
    assert np.abs(g2.sum(axis=0)).max() < 1e-10 * max(1.0, np.abs(g2).max())


def test_full_batch_descent_is_monotone():
    x, xn, W, b, W1, W2 = _problem(7, N=64, scale=0.3, drift=0.5)
    m1, m2 = W1.copy(), W2.copy()
    prev = None
    for _ in range(100):
        loss, g1, g2, _ = O.distill_grads(x, xn, W, b, m1, m2, round_activation=False)
        if prev is not None:
            assert loss < prev
        prev = loss
        m1, _ = O.distill_apply(m1, g1, 0.05, x.shape[0])
        m2, _ = O.distill_apply(m2, g2, 0.05, x.shape[0])


def test_apply_rounds_master_to_bf16():
    m = np.array([[1.0, -2.0], [0.5, 3.0]])
    g = np.array([[2.0 ** -9 * 4, 0.0], [0.0, 1.0]])
    m2, w = O.distill_apply(m, g, lr=1.0, n_total=4)        # step = g / 4
    assert np.array_equal(m2, m - g / 4)
    assert w[0, 0] == 1.0          # 1 − 2⁻⁹ is the midpoint of 1 − 2⁻⁸ and 1: ties to even
    assert w[1, 1] == 2.75


def test_fidelity_spec_examples():
    # identical → (1, 1, 1); disjoint with k < E/2 → (0, 0, 0)
    r = np.random.default_rng(0)
    l = r.normal(size=(50, 16))
    assert O.fidelity_metrics(l, l, 4) == (1.0, 1.0, 1.0)
    t = np.zeros((1, 16))
    t[0, :4] = [4, 3, 2, 1]          # true top-4 = {0,1,2,3}
    p = np.zeros((1, 16))
    p[0, 8:16] = np.arange(8, 0, -1)  # predicted top-8 ⊂ {8..15}
    assert O.fidelity_metrics(p, t, 4) == (0.0, 0.0, 0.0)
    # SPEC S:407-412 tie rule inside the sets: all-equal logits → {0, 1}
    assert O.topk_ids(np.zeros((1, 4)), 2).tolist() == [[0, 1]]


def test_fidelity_hand_example():
    # true order 0 > 1 > 2 > 3 > ...; predicted order 1 > 4 > 0 > 5 > 2 > ...
    t = np.array([[9, 8, 7, 6, 0, 0, 0, 0]], float)
    p = np.array([[7, 9, 5, 0, 8, 6, 0, 0]], float)
    hit, half, rec = O.fidelity_counts(p, t, 3)
    # S={0,1,2}, P={1,4,0}: |S∩P| = 2; S^2={0,1} ⊂ P → 2; P^6={1,4,0,5,2,3} ⊇ S → 3
    assert (hit, half, rec) == (2, 2, 3)


def test_fidelity_recall_dominates_accuracy_brute_force():
    r = np.random.default_rng(9)
    for _ in range(20):
        E, k = int(r.choice([8, 16, 32])), int(r.integers(1, 5))
        t, p = r.normal(size=(30, E)), r.normal(size=(30, E))
        acc, half, rec = O.fidelity_metrics(p, t, k)
        assert rec >= acc
        # brute force: rank positions by explicit sort of (−logit, id) pairs
        hits = 0
        for i in range(30):
            st = sorted(range(E), key=lambda e: (-t[i, e], e))[:k]
            sp = sorted(range(E), key=lambda e: (-p[i, e], e))[:k]
            hits += len(set(st) & set(sp))
        assert hits == round(acc * 30 * k)

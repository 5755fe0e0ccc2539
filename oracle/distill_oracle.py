"""Scale-driven online distillation of the lookahead predictor (NEXT-1) — fp64 CPU oracle.

TEST INFRASTRUCTURE ONLY (same rules as probe_oracle.py: imported solely by tests/,
__graft_entry__.smoke() and bench.py's oracle legs; shares no code with the CUDA path).

P:387-390 "By minimizing the Cross-Entropy loss between the predictor's output and the
ground-truth router's probability distribution, we force the lightweight MLP to align its
trajectory with the actual gating logic" — the frozen prior W_L, b_L is not trained
("pre-trained router as a strong prior"), only the residual Ŵ¹, Ŵ² (Eq. (P)).

Readings (R33-R37):
  R33  teacher p_t = softmax(W_L x^{(L)}_t + b_L): the ground-truth router of layer L on the
       hidden state that actually enters layer L; student q_t = softmax(l̂_t) with
       l̂_t = W_L x^{(L-1)}_t + b_L + Ŵ² bf16(σ(Ŵ¹ x^{(L-1)}_t))  (Eq. (P), R8).
  R34  loss = Σ_t CE(p_t, q_t) = Σ_t [logsumexp(l̂_t) − Σ_e p_te l̂_te]; gradients are those
       of this SUM (so shards all-reduce by SUM and divide by the global token count).
  R35  the bf16 rounding of the activation is the identity in the backward pass (straight
       through); σ'(z) = σ(z)(1 + z(1 − σ(z))) on the unrounded pre-activation z.
  R36  one step is plain gradient descent on fp32 master weights:
       Ŵ ← Ŵ − (lr / N_total) ∇Ŵ, and the product path uses bf16(Ŵ).
  R37  fidelity: top-K accuracy = |S_t ∩ P_t| / k averaged,
       top-half-K hit = |S_t^{⌈k/2⌉} ∩ P_t| / ⌈k/2⌉, 2×top-K recall = |S_t ∩ P_t^{2k}| / k,
       S = teacher top-k, P = predicted top-k, sets by (logit ↓, id ↑).

Pins: tests/test_oracle_distill.py (central finite differences, torch.autograd fp64 as
an independent backprop, Gibbs' inequality, zero-residual closed forms, column sums of
the softmax Jacobian, monotone full-batch descent, SPEC fidelity examples, brute force).
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np

from .probe_oracle import round_bf16, router_logits, silu, topk_ids

__all__ = ["softmax", "silu_grad", "distill_forward", "distill_loss", "distill_grads",
           "distill_apply", "fidelity_counts", "fidelity_metrics"]


def softmax(l: np.ndarray) -> np.ndarray:
    l = np.asarray(l, np.float64)
    m = l.max(axis=1, keepdims=True)
    e = np.exp(l - m)
    return e / e.sum(axis=1, keepdims=True)


def _logsumexp(l: np.ndarray) -> np.ndarray:
    m = l.max(axis=1)
    return m + np.log(np.exp(l - m[:, None]).sum(axis=1))


def silu_grad(z: np.ndarray) -> np.ndarray:
    """d/dz [z σ(z)] = σ(z) (1 + z (1 − σ(z)))   (R35)."""
    s = 1.0 / (1.0 + np.exp(-np.asarray(z, np.float64)))
    return s * (1.0 + z * (1.0 - s))


def distill_forward(x, x_next, W, b, W1, W2, round_activation: bool = True) -> Dict[str, np.ndarray]:
    """Student and teacher logits plus the intermediates the backward pass needs (R33)."""
    x = np.asarray(x, np.float64)
    z = x @ np.asarray(W1, np.float64).T                       # Ŵ¹ x
    a = silu(z)
    if round_activation:
        a = round_bf16(a)                                       # R8
    lhat = router_logits(x, W, b) + a @ np.asarray(W2, np.float64).T      # Eq. (P)
    t = router_logits(x_next, W, b)                             # ground-truth router (R33)
    return {"z": z, "a": a, "lhat": lhat, "t": t}


def distill_loss(x, x_next, W, b, W1, W2, round_activation: bool = True) -> float:
    """Σ_t CE(softmax(t_t), softmax(l̂_t))   (R34)."""
    f = distill_forward(x, x_next, W, b, W1, W2, round_activation)
    p = softmax(f["t"])
    return float(np.sum(_logsumexp(f["lhat"]) - np.sum(p * f["lhat"], axis=1)))


def distill_grads(x, x_next, W, b, W1, W2, round_activation: bool = True
                  ) -> Tuple[float, np.ndarray, np.ndarray, Dict[str, np.ndarray]]:
    """Loss and ∂loss/∂Ŵ¹ [h,H], ∂loss/∂Ŵ² [E,h] by the chain rule (R34, R35):

        g_l = q − p                          ∂CE/∂l̂ for softmax + cross-entropy
        ∇Ŵ² = g_lᵀ a                        l̂ = … + a Ŵ²ᵀ
        g_a = g_l Ŵ²,  g_z = g_a ⊙ σ'(z)     a = σ(z)
        ∇Ŵ¹ = g_zᵀ x                        z = x Ŵ¹ᵀ
    """
    f = distill_forward(x, x_next, W, b, W1, W2, round_activation)
    p, q = softmax(f["t"]), softmax(f["lhat"])
    loss = float(np.sum(_logsumexp(f["lhat"]) - np.sum(p * f["lhat"], axis=1)))
    gl = q - p
    gW2 = gl.T @ f["a"]
    ga = gl @ np.asarray(W2, np.float64)
    gz = ga * silu_grad(f["z"])
    gW1 = gz.T @ np.asarray(x, np.float64)
    f.update(p=p, q=q, gl=gl)
    return loss, gW1, gW2, f


def distill_apply(master: np.ndarray, grad: np.ndarray, lr: float, n_total: int):
    """R36: Ŵ ← Ŵ − (lr / N) ∇Ŵ on the master copy; returns (master', bf16(master'))."""
    m = np.asarray(master, np.float64) - (lr / n_total) * np.asarray(grad, np.float64)
    return m, round_bf16(m)


def fidelity_counts(pred_logits: np.ndarray, true_logits: np.ndarray, k: int) -> Tuple[int, int, int]:
    """Integer hit counts behind R37's three metrics, summed over tokens:
    (Σ|S∩P|, Σ|S^{⌈k/2⌉}∩P|, Σ|S∩P^{2k}|)."""
    S = topk_ids(true_logits, k)
    kh = (k + 1) // 2
    E = np.asarray(pred_logits).shape[1]
    P2 = topk_ids(pred_logits, min(2 * k, E))
    P = P2[:, :k]
    hit = half = rec = 0
    for t in range(S.shape[0]):
        ps, p2 = set(P[t].tolist()), set(P2[t].tolist())
        hit += sum(int(e) in ps for e in S[t])
        half += sum(int(e) in ps for e in S[t, :kh])
        rec += sum(int(e) in p2 for e in S[t])
    return hit, half, rec


def fidelity_metrics(pred_logits, true_logits, k: int) -> Tuple[float, float, float]:
    """(top-K accuracy, top-half-K hit rate, 2×top-K recall)   (R37)."""
    n = np.asarray(true_logits).shape[0]
    hit, half, rec = fidelity_counts(pred_logits, true_logits, k)
    return hit / (n * k), half / (n * ((k + 1) // 2)), rec / (n * k)

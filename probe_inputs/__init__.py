"""Seeded synthetic inputs for the PROBE MoE hot path (shared by the CUDA path's
tests/bench AND the fp64 oracle).

This module holds NONE of the method's arithmetic: no gating, no top-k, no
softmax, no planning, no expert FFN.  It only draws random numbers and builds
tensors whose values are exactly representable in bf16 ("input
recipe"; SURVEY.md §8(d) "Hadamard-encoded routing").

Workload shape (paper): Zipf-skewed expert popularity whose hotspots migrate
step to step (§2.1 "Characterizing Expert Load Imbalance";
BASELINE.json configs[4]); per-rank token batches (chunked prefill per
rank); next-layer prediction accuracy ~0.9 (§4.2).

Construction ("Hadamard encoding").  With n_h a power of two and Had the
Sylvester Hadamard matrix of order n_h:
  * router of layer parity p:   W_p[e, :n_h] = 2^-4 * Had[p*E + e],  zeros beyond n_h
  * token x_t[:n_h] = n_h^-1 * ( sum_j v_j Had[p*E + S_tj]
                                + sum_j v_j Had[(1-p)*E + P_tj]
                                + sum_{4 noise rows >= 2E} nu Had[row] )
  * x_t[n_h:] = bf16(0.05 N(0,1))
so that <x_t, W_p[e]> = v_j/16 if e == S_tj else 0, exactly, in any fp32 order.
S_t is the designed routing of the current layer, P_t the designed prediction of
the next layer's routing (S'_t with each slot replaced with prob. 1-a).
Numerators v = (16, 15, ..., 17-k).  1/32 of tokens get an in-set tied pair of
numerators and 1/32 an extra out-of-set expert tied with slot k (these pin the
tie rules; the expected routing is derived in tests, not here).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import List, Optional

import numpy as np
import torch

MASTER_SEED = 20260217

# ----------------------------------------------------------------------------
# Shapes (BASELINE.json configs).  T is tokens PER RANK.
# ----------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class MoEShape:
    name: str
    E: int      # experts
    k: int      # top-k
    H: int      # hidden
    F: int      # expert ffn width
    T: int      # tokens per rank
    G: int      # EP ranks
    h: int = 0  # predictor residual width (paper silent; default H/4)

    def __post_init__(self):
        if self.h == 0:
            object.__setattr__(self, "h", self.H // 4)

    def with_(self, **kw) -> "MoEShape":
        return dataclasses.replace(self, **kw)

    @property
    def n_h(self) -> int:
        """Largest power of two <= H with n_h >= 2E + 8."""
        n = 1 << int(math.floor(math.log2(self.H)))
        if n < 2 * self.E + 8:
            raise ValueError(f"H={self.H} too small for Hadamard encoding of E={self.E}")
        return n


C0 = MoEShape("C0", E=8, k=2, H=256, F=512, T=64, G=2)
C1 = MoEShape("C1", E=128, k=8, H=2048, F=768, T=8192, G=8)
C2 = MoEShape("C2", E=128, k=4, H=2880, F=2880, T=256, G=8)
C3 = MoEShape("C3", E=256, k=8, H=7168, F=2048, T=16384, G=8)
SHAPES = {s.name: s for s in (C0, C1, C2, C3)}


# ----------------------------------------------------------------------------
# Seeds: sub-seed = SHA-256(master, cfg, step, layer, rank, purpose)
# ----------------------------------------------------------------------------

def sub_seed(*parts) -> int:
    h = hashlib.sha256(repr((MASTER_SEED,) + tuple(parts)).encode()).digest()
    return int.from_bytes(h[:8], "little")


def rng(*parts) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(sub_seed(*parts)))


def torch_gen(*parts) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(sub_seed(*parts) & ((1 << 63) - 1))
    return g


# ----------------------------------------------------------------------------
# Hadamard
# ----------------------------------------------------------------------------

def hadamard_rows(n: int, rows: np.ndarray) -> np.ndarray:
    """Rows of the Sylvester Hadamard matrix of order n: Had[i, j] = (-1)^popcount(i & j)."""
    rows = np.asarray(rows, dtype=np.int64)
    j = np.arange(n, dtype=np.int64)
    a = rows.reshape(-1, 1) & j.reshape(1, -1)
    par = np.zeros_like(a)
    while np.any(a):
        par ^= a & 1
        a >>= 1
    return (1 - 2 * par).astype(np.int8).reshape(rows.shape + (n,))


# ----------------------------------------------------------------------------
# Routing designs
# ----------------------------------------------------------------------------

def zipf_popularity(E: int, s: float, perm: np.ndarray) -> np.ndarray:
    """p_i ∝ i^-s (i = 1..E), assigned to experts through a permutation."""
    base = np.arange(1, E + 1, dtype=np.float64) ** (-s)
    base /= base.sum()
    pop = np.empty(E)
    pop[perm] = base
    return pop


@dataclasses.dataclass
class RankDesign:
    S: np.ndarray        # [T,k] designed routing of this layer (draw order, hottest key first)
    numer: np.ndarray    # [T,k] numerators v_j assigned to S slots
    tie_e: np.ndarray    # [T] extra out-of-set expert tied with slot k (-1 none)
    P: np.ndarray        # [T,k] designed prediction of the NEXT layer's routing
    S_next: np.ndarray   # [T,k] next layer's designed routing (what P approximates)
    noise_rows: np.ndarray  # [T,4]
    noise_coef: np.ndarray  # [T,4]


def draw_routing(shape: MoEShape, step: int, layer: int, rank: int, zipf_s: float,
                 hot_period: int = 1, perm_key=None) -> np.ndarray:
    """Gumbel-top-k (without replacement) of log popularity; the popularity
    permutation is redrawn every `hot_period` steps (hotspot migration).  `perm_key`
    fixes the permutation independently of (step, layer) (stationary hotspots)."""
    E, k, T = shape.E, shape.k, shape.T
    if perm_key is None:
        perm = rng(shape.name, step // hot_period, layer, "perm", zipf_s).permutation(E)
    else:
        perm = rng(shape.name, "perm-key", perm_key, zipf_s).permutation(E)
    pop = zipf_popularity(E, zipf_s, perm)
    g = rng(shape.name, step, layer, rank, "gumbel", zipf_s).gumbel(size=(T, E))
    key = np.log(pop)[None, :] + g
    order = np.argsort(-key, axis=1, kind="stable")[:, :k]
    return order.astype(np.int64)


def design_rank(shape: MoEShape, step: int, layer: int, rank: int, zipf_s: float,
                accuracy: float, hot_period: int = 1, ties: bool = True,
                wrap: Optional[int] = None, perm_key=None) -> RankDesign:
    """wrap: layers form a cycle of this length (layer L's "next layer" is (L+1) mod wrap)."""
    E, k, T = shape.E, shape.k, shape.T
    S = draw_routing(shape, step, layer, rank, zipf_s, hot_period, perm_key)
    nxt = layer + 1 if wrap is None else (layer + 1) % wrap
    S_next = draw_routing(shape, step, nxt, rank, zipf_s, hot_period, perm_key)
    r = rng(shape.name, step, layer, rank, "design", zipf_s, accuracy)
    numer = np.tile(np.arange(16, 16 - k, -1, dtype=np.int64), (T, 1))
    tie_e = np.full(T, -1, dtype=np.int64)
    if ties and k >= 2:
        u = r.random(T)
        in_set = u < 1.0 / 32
        boundary = (u >= 1.0 / 32) & (u < 2.0 / 32)
        for t in np.nonzero(in_set)[0]:
            j = int(r.integers(0, k - 1))
            numer[t, j + 1] = numer[t, j]
        for t in np.nonzero(boundary)[0] if k < E else ():   # k = E: no expert outside the set
            cand = np.setdiff1d(np.arange(E), S[t])
            tie_e[t] = int(cand[r.integers(0, len(cand))])
    # prediction: each slot of S_next kept with prob `accuracy`, else a uniform
    # expert outside S_next ∪ P ("≈90% Top-K accuracy"); rejection sampling,
    # vectorised over tokens, slots in order.
    P = S_next.copy()
    for j in range(k):
        rep = r.random(T) >= accuracy
        idx = np.nonzero(rep)[0]
        # degenerate 2k >= E: a token whose S_next ∪ P already covers every expert keeps its slot
        full = np.array([len(np.union1d(S_next[t], P[t])) >= E for t in idx], dtype=bool)
        idx = idx[~full]
        while len(idx):
            cand = r.integers(0, E, size=len(idx))
            bad = (cand[:, None] == S_next[idx]).any(axis=1) | (cand[:, None] == P[idx]).any(axis=1)
            ok = idx[~bad]
            P[ok, j] = cand[~bad]
            idx = idx[bad]
    n_h = shape.n_h
    noise_rows = r.integers(2 * E, n_h, size=(T, 4))
    noise_coef = r.integers(-8, 9, size=(T, 4))
    return RankDesign(S, numer, tie_e, P, S_next, noise_rows, noise_coef)


# ----------------------------------------------------------------------------
# Tensors
# ----------------------------------------------------------------------------

def encode_tokens(shape: MoEShape, d: RankDesign, parity: int, step: int, layer: int,
                  rank: int, device="cpu") -> torch.Tensor:
    """x [T,H] bf16 from a design (exact integer accumulation, then /n_h)."""
    E, k, T, H, n_h = shape.E, shape.k, shape.T, shape.H, shape.n_h
    p = parity
    # coefficient matrix rows: (Hadamard row index, integer coefficient)
    idx = [p * E + d.S, (1 - p) * E + d.P, d.noise_rows]
    coef = [d.numer, np.tile(np.arange(16, 16 - k, -1), (T, 1)), d.noise_coef]
    has_tie = d.tie_e >= 0
    tie_row = np.where(has_tie, p * E + np.maximum(d.tie_e, 0), 0)[:, None]
    tie_coef = np.where(has_tie, d.numer[:, k - 1], 0)[:, None]
    idx.append(tie_row)
    coef.append(tie_coef)
    idx = torch.from_numpy(np.concatenate(idx, axis=1)).to(device)
    coef = torch.from_numpy(np.concatenate(coef, axis=1).astype(np.int32)).to(device)
    had = torch.from_numpy(hadamard_rows(n_h, np.arange(n_h)).astype(np.int32)).to(device)
    acc = torch.zeros(T, n_h, dtype=torch.int32, device=device)
    for j in range(idx.shape[1]):
        acc += coef[:, j:j + 1] * had[idx[:, j]]
    if int(acc.abs().max()) > 256:
        raise AssertionError("encoded numerator sum exceeds bf16's exact-integer range")
    x = torch.empty(T, H, dtype=torch.bfloat16, device=device)
    x[:, :n_h] = (acc.to(torch.float32) / n_h).to(torch.bfloat16)
    if H > n_h:
        noise = torch.randn(T, H - n_h, generator=torch_gen(shape.name, step, layer, rank, "xtail"))
        x[:, n_h:] = (0.05 * noise).to(torch.bfloat16).to(device)
    # every entry must round-trip exactly (acc/n_h is exact by the range check)
    return x


def router_weight(shape: MoEShape, parity: int, device="cpu") -> torch.Tensor:
    E, H, n_h = shape.E, shape.H, shape.n_h
    w = torch.zeros(E, H, dtype=torch.float32)
    w[:, :n_h] = torch.from_numpy(hadamard_rows(n_h, parity * E + np.arange(E)).astype(np.float32)) / 16.0
    return w.to(torch.bfloat16).to(device)


def expert_weights(shape: MoEShape, parity: int, experts=None, device="cpu", dtype=torch.bfloat16):
    """W13 [E,2F,H] (gate rows 0..F-1, up rows F..2F-1) and W2 [E,H,F], N(0,1)/sqrt(fan_in) stored
    in `dtype` (bf16: rounded; fp32: the full fp32 draw, for the fp32 parity path)."""
    E, H, F = shape.E, shape.H, shape.F
    experts = range(E) if experts is None else experts
    w13 = torch.empty(len(experts), 2 * F, H, dtype=dtype)
    w2 = torch.empty(len(experts), H, F, dtype=dtype)
    for i, e in enumerate(experts):
        g = torch_gen(shape.name, parity, int(e), "experts")
        w13[i] = (torch.randn(2 * F, H, generator=g) / math.sqrt(H)).to(dtype)
        w2[i] = (torch.randn(H, F, generator=g) / math.sqrt(F)).to(dtype)
    return w13.to(device), w2.to(device)


def predictor_residual(shape: MoEShape, parity: int, zero: bool = False, device="cpu"):
    """Ŵ1 [h,H] = bf16(N(0,1)/sqrt(H)); Ŵ2 [E,h] scaled so ||Ŵ2 a||_inf < 2^-6 for |a| <= max SiLU range.

    The bound uses |a_i| <= |z_i| + 1 with |z| <= ||Ŵ1||_row,1 * ||x||_inf; we simply scale
    Ŵ2 so that sum_i |Ŵ2[e,i]| * A_max < 2^-6 where A_max bounds |a| (checked at use by tests).
    """
    E, H, h = shape.E, shape.H, shape.h
    g = torch_gen(shape.name, parity, "residual")
    w1 = (torch.randn(h, H, generator=g) / math.sqrt(H)).to(torch.bfloat16)
    w2 = torch.randn(E, h, generator=g)
    if zero:
        w2 = torch.zeros(E, h)
    else:
        # |x| <= 256/n_h + tail; |z_i| <= sum_h |w1| * max|x|
        xmax = 256.0 / shape.n_h + (0.05 * 6.0 if shape.H > shape.n_h else 0.0)
        zmax = float(w1.float().abs().sum(dim=1).max()) * xmax
        amax = zmax + 1.0
        row1 = float(w2.abs().sum(dim=1).max())
        scale = (2.0 ** -6) / (row1 * amax) * 0.5
        # keep it a power of two so the bf16 values stay "nice"
        scale = 2.0 ** math.floor(math.log2(scale))
        w2 = w2 * scale
    return w1.to(device), w2.to(torch.bfloat16).to(device)


def predictor_residual_relabel(shape: MoEShape, parity: int, frac: float = 0.25, device="cpu"):
    """A residual large enough to CHANGE the predicted top-k sets, with every value exact.

    For a seeded expert set D (|D| = max(2, round(frac·E)), at most h) and the cyclic shift
    σ on D:  Ŵ1[j, :n_h] = 2·Had[parity·E + D_j] (zeros elsewhere, rows j >= |D| zero) and
    Ŵ2[σ(D_j), j] = +2^-5, Ŵ2[D_j, j] = -2^-5.  On an encoded token the product Ŵ1 x reads
    the designed integer coefficient of each D_j exactly (0 or a numerator 17-k..16), so the
    activation is 0 or a value far from any bf16 rounding boundary, and Ŵ2 a moves the prior
    coefficient of D_j onto σ(D_j): the predicted set becomes P_t relabelled on D, in
    multiples of 1/16 (exact in fp32 in any order).  Only random draws and fixed tensor
    construction here; the expected counts come from the oracle."""
    E, H, h, n_h = shape.E, shape.H, shape.h, shape.n_h
    m = min(h, max(2, int(round(frac * E))))
    D = np.sort(rng(shape.name, parity, "relabel-set", frac).choice(E, size=m, replace=False))
    sig = np.roll(D, -1)
    w1 = torch.zeros(h, H, dtype=torch.float32)
    w1[:m, :n_h] = 2.0 * torch.from_numpy(hadamard_rows(n_h, parity * E + D).astype(np.float32))
    w2 = torch.zeros(E, h, dtype=torch.float32)
    j = torch.arange(m)
    w2[torch.from_numpy(sig), j] = 2.0 ** -5
    w2[torch.from_numpy(D), j] = -(2.0 ** -5)
    return w1.to(torch.bfloat16).to(device), w2.to(torch.bfloat16).to(device)


@dataclasses.dataclass
class LayerInputs:
    layer: int
    parity: int
    x: torch.Tensor            # [G_loc, T, H] bf16 for the requested ranks
    designs: List[RankDesign]  # per requested rank


def layer_inputs(shape: MoEShape, step: int, layer: int, zipf_s: float = 1.0,
                 accuracy: float = 0.9, ranks: Optional[List[int]] = None, device="cpu",
                 hot_period: int = 1, ties: bool = True, wrap: Optional[int] = None,
                 perm_key=None) -> LayerInputs:
    ranks = list(range(shape.G)) if ranks is None else ranks
    p = layer % 2
    xs, ds = [], []
    for r in ranks:
        d = design_rank(shape, step, layer, r, zipf_s, accuracy, hot_period, ties, wrap, perm_key)
        xs.append(encode_tokens(shape, d, p, step, layer, r, device))
        ds.append(d)
    return LayerInputs(layer, p, torch.stack(xs), ds)


# ----------------------------------------------------------------------------
# Secondary "natural" generator: 5-bit dyadic grid; logits are
# exact in fp32 and integer-valued ties are frequent (exercise tie rules).
# ----------------------------------------------------------------------------

def dyadic(shape_, *seed_parts, lim=32, scale=2.0 ** -4, device="cpu"):
    r = rng(*seed_parts)
    v = r.integers(-lim, lim + 1, size=shape_).astype(np.float32) * scale
    return torch.from_numpy(v).to(torch.bfloat16).to(device)


NATURAL_SCALE = 2.0 ** -6     # x and router entries: integers in [-32, 32] times 2^-6


def natural_router(shape: MoEShape, layer: int, step: int = 0, zipf_s: float = 1.2, beta: float = 1.0,
                   dup_frac: float = 0.125, device="cpu"):
    """Router W [E,H] bf16 and bias b [E] fp32 of the "natural" generator.

    W on the 5-bit dyadic grid (|i| <= 32, scale 2^-6); a seeded dup_frac of the experts
    copy the row (and bias) of a lower-id expert, so exact logit ties occur whenever both
    are in contention (pins the lowest-id rule, R3).  Skew: dyadic bias
    b_e = round_{2^-4}(beta · log p_{π(e)}) with the Zipf popularity permuted per
    (step, layer) (hotspot migration).  Logits x·Wᵀ + b are exact in fp32 in any order:
    products are multiples of 2^-12 and |ℓ| < 2^(log2(H)-2) + 8, inside 24 bits."""
    E, H = shape.E, shape.H
    W = dyadic((E, H), shape.name, layer % 2, "natural-router", scale=NATURAL_SCALE).float()
    perm = rng(shape.name, step, layer, "natural-perm", zipf_s).permutation(E)
    pop = zipf_popularity(E, zipf_s, perm)
    b = np.round(beta * np.log(pop) * 16.0) / 16.0
    r = rng(shape.name, layer % 2, "natural-dups")
    ndup = int(round(dup_frac * E))
    dups = r.choice(np.arange(1, E), size=ndup, replace=False)
    for e in np.sort(dups):
        src = int(r.integers(0, e))
        W[e] = W[src]
        b[e] = b[src]
    return W.to(torch.bfloat16).to(device), torch.from_numpy(b.astype(np.float32)).to(device)


def natural_layer_inputs(shape: MoEShape, step: int, layer: int, ranks: Optional[List[int]] = None,
                         device="cpu") -> "LayerInputs":
    """Tokens of the natural generator: x [G,T,H] on the 5-bit dyadic grid (scale 2^-6),
    i.i.d. per (step, layer, rank); routing is whatever the router and bias make of it
    (negative and dense logits, exact ties from duplicated router rows)."""
    ranks = list(range(shape.G)) if ranks is None else ranks
    xs = [dyadic((shape.T, shape.H), shape.name, step, layer, r, "natural-x", scale=NATURAL_SCALE, device=device)
          for r in ranks]
    return LayerInputs(layer, layer % 2, torch.stack(xs), [])


def bf16_to_numpy_f64(t: torch.Tensor) -> np.ndarray:
    """Exact decode of a bf16 tensor to float64 numpy (bit manipulation only)."""
    bits = t.detach().cpu().contiguous().view(torch.int16).numpy().astype(np.uint16).astype(np.uint32)
    return (bits << 16).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------
# Distillation task: "feature drift" between adjacent layers
# ----------------------------------------------------------------------------

@dataclasses.dataclass
class DistillTask:
    x: torch.Tensor        # [G, T, H] bf16: the hidden state the predictor reads
    x_next: torch.Tensor   # [G, T, H] bf16: the hidden state the teacher router reads
    W: torch.Tensor        # [E, H] bf16: the frozen router of the predicted layer
    drifted: np.ndarray    # experts whose routing mass the drift relabels


def distill_task(shape: MoEShape, step: int, zipf_s: float = 1.2, drift_frac: float = 0.35,
                 router_scale: float = 4.0, device="cpu") -> DistillTask:
    """x = layer-0 inputs (whose parity-1 encoding is the prior's prediction P_t); x_next = x
    plus a fixed linear drift that moves the parity-1 coefficient of every expert e in a
    seeded set D (|D| = drift_frac·E) onto the next expert of D (cyclic), so the teacher's
    top-k is P_t relabelled on D: the frozen prior misses those slots (the "untrained"
    accuracy) and a residual that learns the relabelling recovers them.  The router
    is the parity-1 router scaled by `router_scale` (a power of two: exact in bf16), which
    sharpens the teacher distribution without changing any top-k set."""
    E, n_h = shape.E, shape.n_h
    li = layer_inputs(shape, step, 0, zipf_s, accuracy=1.0, device=device)
    D = np.sort(rng(shape.name, "drift-set").choice(E, size=max(2, int(round(drift_frac * E))), replace=False))
    pi = np.roll(D, -1)
    Hd = torch.from_numpy(hadamard_rows(n_h, E + D).astype(np.float32)).to(device)
    Hp = torch.from_numpy(hadamard_rows(n_h, E + pi).astype(np.float32)).to(device)
    xf = li.x.float()
    coef = xf[..., :n_h] @ Hd.T                       # ⟨x, h_{E+e}⟩ (exact small integers)
    xn = li.x.clone()
    xn[..., :n_h] = (xf[..., :n_h] + coef @ (Hp - Hd) / n_h).to(torch.bfloat16)
    W = (router_weight(shape, 1).float() * router_scale).to(torch.bfloat16).to(device)
    return DistillTask(li.x, xn, W, D)

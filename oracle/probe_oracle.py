"""PROBE MoE hot path — plain, slow, fp64 CPU oracle.

TEST INFRASTRUCTURE ONLY.  Imported solely by tests/, __graft_entry__.smoke()
and bench.py (cpu_baseline / --impl reference).  Shares no code with the CUDA
path (paper_2602_00509_b200/), and the CUDA path never imports it.

Every function follows the paper (PAPER.md, cited as P:<line>) in the paper's
order and notation; where the paper is silent or ambiguous the reading from
SURVEY.md §8(c) (R1..R32, listed in DESIGN.md §2) is used.  Floating point is
fp64 on the bf16-decoded inputs; the one declared rounding point is the
predictor's residual activation (R8).  Integer steps (routing ids, counts,
plans, splits, layouts) use Python / numpy int64.

Pins (tests/test_oracle_*.py): SPEC worked examples (S:127-128, S:157-158,
S:177-178, S:313/325/334),
Hadamard-encoded designed routing, closed forms (softmax sums to 1, Ŵ2 = 0
prior, x = 0 bias, dense SwiGLU), brute-force Eq. 7 optimum (scipy MILP) on
tiny instances, conservation/validity invariants.  No function is
"parity unpinned".
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "round_bf16", "router_logits", "topk_ids", "gate", "silu", "predictor_logits",
    "predict_counts", "PlannerConfig", "Plan", "replica_caps", "rank_costs",
    "token_loads", "plan_greedy", "static_plan", "materialize", "slot_experts",
    "dispatch_layout", "Layout", "swiglu_expert", "combine", "moe_layer_outputs", "moe_outputs_ranks",
    "imbalance_ratio", "expert_compute_time", "traffic_volumes", "transfer_latency",
    "exposed_overhead", "replica_slot_schedule", "layer_reference",
]


# =============================================================================
# numerics helpers
# =============================================================================

def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16 (8 significant bits), returned as float64.

    Direct from fp64 (no fp32 intermediate): a = m * 2^e with m in [0.5, 1);
    keep 8 bits of m, ties to even (np.rint).  Normal range only (enough here).
    """
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)
    return np.ldexp(np.rint(np.ldexp(m, 8)), e - 8)


# =============================================================================
# a1 — gate (ground-truth router), "standard sequence of MoE operators",
#      P:385 "actual token dispatch strictly follows the ground-truth router"
# =============================================================================

def router_logits(x: np.ndarray, W: np.ndarray, b: Optional[np.ndarray] = None) -> np.ndarray:
    """ℓ_{t,e} = Σ_h x_{t,h} W_{e,h} + b_e   (frozen prior term W_L h + b_L)."""
    l = np.asarray(x, np.float64) @ np.asarray(W, np.float64).T
    if b is not None:
        l = l + np.asarray(b, np.float64)[None, :]
    return l


def topk_ids(logits: np.ndarray, k: int) -> np.ndarray:
    """First k experts by (logit ↓, expert id ↑)   (R3 lowest-id ties, R4 slot order)."""
    order = np.argsort(-np.asarray(logits, np.float64), axis=1, kind="stable")
    return order[:, :k].astype(np.int64)


def gate(x, W, b, k):
    """Top-k routing with softmax over the k selected logits (R1).

    Returns ids [T,k] (slot order), weights g [T,k] (fp64), counts n[e] = |{t: e ∈ S_t}|.
    """
    l = router_logits(x, W, b)
    ids = topk_ids(l, k)
    sel = np.take_along_axis(l, ids, axis=1)
    m = sel.max(axis=1, keepdims=True)
    w = np.exp(sel - m)
    g = w / w.sum(axis=1, keepdims=True)
    counts = np.bincount(ids.reshape(-1), minlength=W.shape[0]).astype(np.int64)
    return ids, g, counts


# =============================================================================
# a2 — Gate-Initialized Lookahead Predictor, Eq. (P)
#      l̂_L = W_L h_{L−1} + b_L + Ŵ²_L σ(Ŵ¹_L h_{L−1}),  σ = SiLU
# =============================================================================

def silu(z: np.ndarray) -> np.ndarray:
    return z / (1.0 + np.exp(-z))


def predictor_logits(x, W_next, b_next, W1, W2, round_activation: bool = True):
    """Eq. (P).  The residual activation a = σ(Ŵ¹x) is rounded to bf16 (R8, declared
    rounding point of this build); everything else fp64.  Returns (l̂, a)."""
    x = np.asarray(x, np.float64)
    prior = router_logits(x, W_next, b_next)
    if W1 is None or W2 is None:
        return prior, None
    z = x @ np.asarray(W1, np.float64).T
    a = silu(z)
    if round_activation:
        a = round_bf16(a)
    return prior + a @ np.asarray(W2, np.float64).T, a


def predict_counts(x, W_next, b_next, W1, W2, k):
    """n̂_r[e] = #tokens on r whose predicted top-k set contains e  (R9)."""
    l, _ = predictor_logits(x, W_next, b_next, W1, W2)
    ids = topk_ids(l, k)
    return np.bincount(ids.reshape(-1), minlength=np.asarray(W_next).shape[0]).astype(np.int64), ids


# =============================================================================
# a4 — Greedy Balance-Optimal Planning, Algorithm 1 under R10–R22
# =============================================================================

@dataclasses.dataclass(frozen=True)
class PlannerConfig:
    G: int                  # ep
    E: int
    replica_budget: int = 3         # "at most three redundant experts per rank" P:476
    kmax: int = 16                  # "hard cap of k_max = 16 iterations" P:476
    alpha_ps: int = 1               # compute cost per routed pair, ps (Eq. 2 with F̄/F_peak; R11)
    beta_ps: int = 0                # comm cost per remote pair, ps (Eq. 4/5, λ = 1; R11)
    n_sat: int = 0                  # η_g knee in pairs (R11): c(m) = max(m, n_sat) for m > 0
    bw_bytes_per_us: int = 770_000  # BW_net for Eq. 6 caps (bytes/µs)
    expert_bytes: int = 1           # 𝒲 = 6HF bytes (bf16)

    @property
    def EL(self) -> int:
        return self.E // self.G

    def home(self, e: int) -> int:
        return e // self.EL


@dataclasses.dataclass
class Plan:
    replicas: List[List[int]]        # per rank, sorted expert ids (slot order)
    quota: np.ndarray                # [G,E,G] int64 assignment A on n̂
    transfers: List[Tuple[int, int, int]]  # (expert, sender=home, receiver) in acceptance order
    iterations: int
    maxL_before: int
    maxL_after: int
    L_before: List[int]
    L_after: List[int]
    caps: List[int]


def replica_caps(window_ns: Sequence[int], cfg: PlannerConfig) -> List[int]:
    """Eq. (6) + hiding window: a rank can move n experts iff
    n·𝒲/BW_net ≤ T_window  ⇔  n ≤ floor(T_window·BW/𝒲); capped by the budget (R15, R17)."""
    caps = []
    for w in window_ns:
        n = (int(w) * cfg.bw_bytes_per_us) // (cfg.expert_bytes * 1000)
        caps.append(int(min(cfg.replica_budget, n)))
    return caps


def _c(m: int, n_sat: int) -> int:
    """Per-expert compute cost in pairs: Eq. (2) with saturating η_g(n) = min(1, n/n_sat) (R11)."""
    return 0 if m == 0 else max(m, n_sat)


def rank_costs(split: np.ndarray, hosts: List[set], cfg: PlannerConfig) -> List[int]:
    """L_r = α Σ_{e hosted on r} c(m_{e,r}) + β max(in_r, out_r)   (Eq. 7 per-rank objective, R11/R12).

    m_{e,r} = Σ_s split[s][e][r];  in_r = Σ_{s≠r,e} split[s][e][r];  out_r = Σ_{e,t≠r} split[r][e][t].
    """
    G = cfg.G
    L = []
    for r in range(G):
        comp = 0
        for e in sorted(hosts[r]):
            comp += _c(int(split[:, e, r].sum()), cfg.n_sat)
        inn = int(split[:, :, r].sum() - split[r, :, r].sum())
        out = int(split[r, :, :].sum() - split[r, :, r].sum())
        L.append(cfg.alpha_ps * comp + cfg.beta_ps * max(inn, out))
    return L


def token_loads(split: np.ndarray) -> List[int]:
    """ℒ_r = Σ_e n_{e,r}  (Eq. 1 loads on the assignment, R32)."""
    return [int(v) for v in split.sum(axis=(0, 1))]


def static_plan(nhat: np.ndarray, cfg: PlannerConfig) -> np.ndarray:
    """Locality-first initialization from n̂ and P′ (Alg. 1 line 2; R22 home(e) = e div (E/G))."""
    G, E = cfg.G, cfg.E
    split = np.zeros((G, E, G), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            split[s, e, cfg.home(e)] = int(nhat[s, e])
    return split


def plan_greedy(nhat: np.ndarray, window_ns: Sequence[int], cfg: PlannerConfig) -> Plan:
    """Algorithm 1, line by line, with readings R13–R21."""
    G, E = cfg.G, cfg.E
    nhat = np.asarray(nhat, dtype=np.int64)
    assert nhat.shape == (G, E) and E % G == 0
    # line 1: Δ^in, Δ^out ← ∅; k ← 0
    delta_in: List[List[int]] = [[] for _ in range(G)]
    n_out = [0] * G                       # |Δ^out_r| as a multiset (R16)
    k = 0
    # line 2: A ← locality-first(n̂, P′)
    split = static_plan(nhat, cfg)
    hosts = [set(range(r * cfg.EL, (r + 1) * cfg.EL)) for r in range(G)]
    # line 3: L ← ComputeLatencies(A)
    L = rank_costs(split, hosts, cfg)
    L_before = list(L)
    caps = replica_caps(window_ns, cfg)
    invalid = set()
    transfers = []
    while True:                                               # line 4
        src = min(range(G), key=lambda r: (-L[r], r))         # line 5: argmax L (lowest r on ties)
        cand = [r for r in range(G) if r != src and (src, r) not in invalid]
        if not cand:                                          # R14: no partner ⇒ stop
            break
        dst = min(cand, key=lambda r: (L[r], r))              # line 6: argmin L (R14)
        # line 7: e* = SelectHeavyExpert(r_src, n̂)  (R13)
        best_e, best_pool = -1, 0
        for e in range(src * cfg.EL, (src + 1) * cfg.EL):
            if e in hosts[dst]:
                continue
            pool = int(split[:, e, src].sum() - split[src, e, src])
            if pool > best_pool:
                best_e, best_pool = e, pool
        if best_e < 0:
            invalid.add((src, dst))
            continue
        # line 8-10: dual-side budget (R15)
        if len(delta_in[dst]) + 1 > caps[dst] or n_out[src] + 1 > caps[src]:
            invalid.add((src, dst))
            continue
        # line 11: WaterFillingRebalance (R18)
        loads = token_loads(split)
        avg_ceil = -(-sum(loads) // G)
        x = min(best_pool, max(0, loads[src] - avg_ceil))
        new_split = split.copy()
        remaining = x
        order = [dst] + [s for s in range(G) if s not in (src, dst)]
        for s in order:
            if remaining == 0:
                break
            mv = min(remaining, int(new_split[s, best_e, src]))
            new_split[s, best_e, src] -= mv
            new_split[s, best_e, dst] += mv
            remaining -= mv
        new_hosts = [set(h) for h in hosts]
        new_hosts[dst].add(best_e)
        newL = rank_costs(new_split, new_hosts, cfg)
        gain = L[src] - max(newL[src], newL[dst])             # R19
        # line 12-14: convergence / budget (ε = 0; R19, R20)
        if gain <= 0 or k >= cfg.kmax:
            break
        # line 15-17: accept
        n_out[src] += 1
        delta_in[dst].append(best_e)
        transfers.append((best_e, src, dst))
        split, hosts, L = new_split, new_hosts, newL
        k += 1
    replicas = [sorted(d) for d in delta_in]                  # line 19: UpdatePlacement
    return Plan(replicas, split, transfers, k, max(L_before), max(L), L_before, list(L), caps)


# =============================================================================
# a5 — Update / materialize the plan onto the actual counts (R23)
# =============================================================================

def _hosts_expert(r: int, e: int, replicas: List[List[int]], EL: int) -> bool:
    return e // EL == r or e in replicas[r]


def materialize(n: np.ndarray, quota: Optional[np.ndarray], replicas: List[List[int]],
                G: int, E: int) -> np.ndarray:
    """split[s][e][t] on the actual counts n [G,E] from the quota A (computed on n̂).

    For each (s,e): Q_t = quota[s][e][t], P = Σ_t Q_t.
      P = 0: all n[s][e] tokens go to s if s hosts e, else to home(e).
      else:  a_t = ⌊n·Q_t/P⌋; the leftover goes to the t with the largest Q_t (lowest t on ties).
    quota=None means static EP (empty plan, every Q = 0 and no replicas).
    """
    EL = E // G
    split = np.zeros((G, E, G), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            cnt = int(n[s, e])
            Q = [0] * G if quota is None else [int(v) for v in quota[s, e]]
            P = sum(Q)
            if P == 0:
                t = s if _hosts_expert(s, e, replicas, EL) else e // EL
                split[s, e, t] = cnt
                continue
            a = [cnt * Q[t] // P for t in range(G)]
            tstar = min(range(G), key=lambda t: (-Q[t], t))
            a[tstar] += cnt - sum(a)
            split[s, e, :] = a
    return split


# =============================================================================
# a6 — Dispatch layout (R24) — rows per destination grouped by local slot
# =============================================================================

def slot_experts(r: int, replicas: List[List[int]], G: int, E: int) -> List[int]:
    """Local slots of rank r: base experts ascending, then replicas in slot order (sorted)."""
    EL = E // G
    return list(range(r * EL, (r + 1) * EL)) + sorted(replicas[r])


@dataclasses.dataclass
class Layout:
    dest: List[np.ndarray]       # per source s: [T_s,k] destination rank of each (token, slot)
    row: List[np.ndarray]        # per source s: [T_s,k] row in the destination's receive buffer
    rows: List[List[Tuple[int, int, int, int]]]  # per dest: (src, token, slot j, local slot) in recv order
    group_sizes: List[List[int]]  # per dest: rows per local slot


def dispatch_layout(ids: List[np.ndarray], split: np.ndarray, replicas: List[List[int]],
                    G: int, E: int) -> Layout:
    """Tokens of s routed to e are taken in ascending token index and fill the
    targets t in ascending order with split[s][e][t] tokens each (R23 step 5);
    on destination r, slot j holds rows ordered by (source ↑, token ↑) (R24)."""
    dest = [np.full(i.shape, -1, dtype=np.int64) for i in ids]
    for s in range(G):
        for e in range(E):
            t_idx, j_idx = np.nonzero(ids[s] == e)       # row-major ⇒ ascending token index
            cum = np.cumsum(split[s, e])                 # targets filled in ascending t
            assert cum[-1] == len(t_idx), "split does not cover the routed tokens"
            p = np.arange(len(t_idx))
            dest[s][t_idx, j_idx] = np.searchsorted(cum, p, side="right")
    rows: List[List[Tuple[int, int, int, int]]] = []
    sizes: List[List[int]] = []
    row = [np.full(i.shape, -1, dtype=np.int64) for i in ids]
    for r in range(G):
        lst = []
        sz = []
        for ls, e in enumerate(slot_experts(r, replicas, G, E)):
            before = len(lst)
            for s in range(G):
                t_idx, j_idx = np.nonzero((ids[s] == e) & (dest[s] == r))   # token ↑
                row[s][t_idx, j_idx] = len(lst) + np.arange(len(t_idx))
                lst.extend((s, int(t), int(j), ls) for t, j in zip(t_idx, j_idx))
            sz.append(len(lst) - before)
        rows.append(lst)
        sizes.append(sz)
    return Layout(dest, row, rows, sizes)


# =============================================================================
# a7 — expert SwiGLU FFN; a8 — gate-weighted combine
# =============================================================================

def swiglu_expert(x: np.ndarray, W13: np.ndarray, W2: np.ndarray) -> np.ndarray:
    """y = (SiLU(x W_gᵀ) ⊙ (x W_uᵀ)) W_dᵀ with W13 = [W_g; W_u] [2F,H], W2 = W_d [H,F]; fp64."""
    F = W13.shape[0] // 2
    x = np.asarray(x, np.float64)
    g = x @ np.asarray(W13[:F], np.float64).T
    u = x @ np.asarray(W13[F:], np.float64).T
    return (silu(g) * u) @ np.asarray(W2, np.float64).T


def combine(g: np.ndarray, y: np.ndarray) -> np.ndarray:
    """out_t = Σ_{j<k} g_{t,j} y_{t,j}, summed in slot order (R4, R25). y: [T,k,H]."""
    out = np.zeros((y.shape[0], y.shape[2]), dtype=np.float64)
    for j in range(y.shape[1]):
        out += g[:, j:j + 1] * y[:, j, :]
    return out


def moe_layer_outputs(x: np.ndarray, ids: np.ndarray, g: np.ndarray,
                      W13: Dict[int, np.ndarray], W2: Dict[int, np.ndarray],
                      tokens: Optional[Sequence[int]] = None) -> np.ndarray:
    """MoE output for the given tokens of one source rank.  Placement independent
    (semantic equivalence): each (token, slot) is computed once by its
    expert's weights, wherever the plan sends it."""
    tokens = range(x.shape[0]) if tokens is None else tokens
    tokens = list(tokens)
    k = ids.shape[1]
    H = x.shape[1]
    y = np.zeros((len(tokens), k, H))
    for e in sorted(set(int(v) for v in ids[tokens].reshape(-1))):
        mask = ids[tokens] == e
        ti, jj = np.nonzero(mask)
        y[ti, jj] = swiglu_expert(x[np.asarray(tokens)[ti]], W13[e], W2[e])
    return combine(g[tokens], y)


def moe_outputs_ranks(xs: List[np.ndarray], ids: List[np.ndarray], gs: List[np.ndarray], W13, W2,
                      tokens: Optional[List[Sequence[int]]] = None) -> List[np.ndarray]:
    """moe_layer_outputs for every source rank at once: loop over experts outermost and
    evaluate each expert once on the rows (token, slot) of ALL ranks routed to it, so its
    weights are read once (W13/W2 may decode on access).  Same arithmetic: every row of
    y_{t,j} = swiglu_expert(x_t) with expert ids[t,j] (rows are independent), then combine
    in slot order (R4, R25)."""
    G = len(xs)
    toks = [np.asarray(list(range(xs[s].shape[0])) if tokens is None else list(tokens[s]), dtype=np.int64)
            for s in range(G)]
    k = ids[0].shape[1]
    H = xs[0].shape[1]
    ys = [np.zeros((len(toks[s]), k, H)) for s in range(G)]
    sub = [ids[s][toks[s]] for s in range(G)]
    experts = sorted(set(int(v) for s in range(G) for v in sub[s].reshape(-1)))
    for e in experts:
        hits = [np.nonzero(sub[s] == e) for s in range(G)]
        rows = np.concatenate([xs[s][toks[s][hits[s][0]]] for s in range(G)], axis=0)
        y = swiglu_expert(rows, W13[e], W2[e])
        o = 0
        for s in range(G):
            ti, jj = hits[s]
            ys[s][ti, jj] = y[o:o + len(ti)]
            o += len(ti)
    return [combine(gs[s][toks[s]], ys[s]) for s in range(G)]


# =============================================================================
# analytical model (§3, Eq. 1–6) — used by tests as pins and by reporting
# =============================================================================

def imbalance_ratio(loads: Sequence[float]) -> float:
    """Eq. (1): IR = max_r ℒ_r / mean_r ℒ_r."""
    loads = np.asarray(loads, dtype=np.float64)
    if loads.sum() <= 0:
        raise ValueError("empty workload")
    return float(loads.max() / loads.mean())


def expert_compute_time(n: int, Fbar: float, Fpeak: float, n_sat: int) -> float:
    """Eq. (2): T = n F̄ / (η_g(n) F_peak) with η_g(n) = min(1, n/n_sat) (R11)."""
    if n == 0:
        return 0.0
    eta = min(1.0, n / n_sat) if n_sat > 0 else 1.0
    return n * Fbar / (eta * Fpeak)


def traffic_volumes(split: np.ndarray, H_bytes: float, lam_in=None, lam_out=None):
    """Eq. (4): V^in_r = (H/λ^in_r) Σ_{r'≠r} Σ_e n^{r'}_{e,r};  V^out_r = (H/λ^out_r) Σ_{e, t≠r} n^r_{e,t}."""
    G = split.shape[0]
    lam_in = [1.0] * G if lam_in is None else lam_in
    lam_out = [1.0] * G if lam_out is None else lam_out
    vin, vout = [], []
    for r in range(G):
        inn = split[:, :, r].sum() - split[r, :, r].sum()
        out = split[r].sum() - split[r, :, r].sum()
        vin.append(H_bytes / lam_in[r] * float(inn))
        vout.append(H_bytes / lam_out[r] * float(out))
    return vin, vout


def transfer_latency(n_in: int, n_out: int, W_bytes: float, bw: float) -> float:
    """Eq. (6): T_trans = max(|Δ^in|, |Δ^out|)·𝒲 / BW_net."""
    return max(n_in, n_out) * W_bytes / bw


def exposed_overhead(trans: Sequence[float], window: Sequence[float]) -> float:
    """§3.4 exposed overhead, rank-wise: max(0, max_r(T_trans,r − T_window,r))  (R28 reading)."""
    return max(0.0, max(t - w for t, w in zip(trans, window)))


def replica_slot_schedule(replicas_per_layer: List[List[List[int]]], budget: int = 3):
    """Double-buffered replica slots: layer L uses bank L mod 2 of 2×budget slots.
    Returns per layer per rank the physical slot ids; raises on a budget violation."""
    out = []
    for L, reps in enumerate(replicas_per_layer):
        layer_slots = []
        for r, rr in enumerate(reps):
            if len(rr) > budget:
                raise ValueError(f"rank {r} layer {L}: {len(rr)} replicas exceed budget {budget}")
            layer_slots.append([(L % 2) * budget + i for i in range(len(rr))])
        out.append(layer_slots)
    return out


# =============================================================================
# whole layer (all G ranks simulated in one process) — §8(c) steps 1..8
# =============================================================================

def layer_reference(xs: List[np.ndarray], W: np.ndarray, b: Optional[np.ndarray], k: int,
                    plan: Optional[Plan], G: int, E: int,
                    W13: Optional[Dict[int, np.ndarray]] = None,
                    W2: Optional[Dict[int, np.ndarray]] = None,
                    tokens: Optional[List[Sequence[int]]] = None,
                    with_layout: bool = True):
    """Gate on every rank → actual counts n [G,E] (all-gather) → materialize plan →
    dispatch layout → (optionally) expert FFN + combine for sampled tokens."""
    ids, gs, counts = [], [], []
    for s in range(G):
        i, g, c = gate(xs[s], W, b, k)
        ids.append(i)
        gs.append(g)
        counts.append(c)
    n = np.stack(counts)
    replicas = plan.replicas if plan is not None else [[] for _ in range(G)]
    quota = plan.quota if plan is not None else None
    split = materialize(n, quota, replicas, G, E)
    lay = dispatch_layout(ids, split, replicas, G, E) if with_layout else None
    outs = None
    if W13 is not None:
        outs = moe_outputs_ranks(xs, ids, gs, W13, W2, tokens)
    return dict(ids=ids, g=gs, n=n, split=split, layout=lay, out=outs, replicas=replicas)

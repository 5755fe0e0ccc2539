"""Run the PROBE layer pipeline on the GPU (through the C-ABI) and the fp64 oracle on
the same seeded inputs; return both for element-wise comparison.

Sequence (Continuous Lookahead Pipelining): forward(L0, static — layer 0
is not predicted, R29) → predict(L1) → plan(L1) → prefetch(L1) → forward(L1, plan).
"""
from __future__ import annotations

import dataclasses
import os
from typing import Optional

import numpy as np
import torch

import oracle as O
import probe_inputs as pi


@dataclasses.dataclass
class CaseCfg:
    shape: pi.MoEShape
    zipf_s: float = 1.2
    step: int = 0
    alpha_ps: int = 1
    beta_ps: int = 0
    n_sat: int = 0
    replica_budget: int = 3
    window_ns: int = 10 ** 9
    bw_bytes_per_us: int = 770_000
    residual: bool = True
    out_fp32: bool = True
    capacity_factor: float = 0.0
    bias: bool = False
    sample_tokens: int = 0          # >0: oracle outputs only for this many tokens per rank
    ep_emulation: bool = False      # partitioned expert GEMMs (single-GPU EP straggler emulation)
    fused_epi_topk: bool = False    # router/predictor top-k in the GEMM epilogue
    pair_gemm: bool = True          # expert GEMMs on CTA pairs (cta_group::2); False → 1-CTA kernel
    dtype: str = "bf16"             # "fp32": parity path (fp32 operands, SIMT fp32 GEMMs, fp32 expert weights)
    max_tokens: int = 0             # >T: context capacity above the T this layer call runs with
    gen: str = "hadamard"           # "natural": 5-bit dyadic x / router, dyadic Zipf bias, duplicated router rows
    residual_kind: str = "bounded"  # "relabel": exact residual that changes the predicted sets (n̂)
    dedup_wire: bool = False        # one wire row per unique (token, dest) + R25 partial-sum combine
    predispatch: bool = False       # NEXT-4: pre-dispatch to predicted experts' home ranks during the gate
    fuse_gate_predictor: bool = False  # gate GEMM of layer 0 also computes layer 1's prior + Ŵ1 activation

    @property
    def es(self) -> int:
        return 4 if self.dtype == "fp32" else 2


def f64(t):
    if t.dtype == torch.float32:
        return t.detach().cpu().double().numpy()
    return pi.bf16_to_numpy_f64(t)


class LazyExperts:
    """Expert weights decoded to fp64 on access, not cached (the oracle reads each expert once
    per layer; at C3 the decoded weights of one parity would take 90 GB)."""

    def __init__(self, w):
        self.w = w

    def __getitem__(self, e):
        return f64(self.w[e])


def run_gpu(case: CaseCfg):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    sh = case.shape
    G, E, k, H, F, T, h = sh.G, sh.E, sh.k, sh.H, sh.F, sh.T, sh.h
    cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=F, T=max(T, case.max_tokens), h=h if case.residual else 0,
                      replica_budget=case.replica_budget, alpha_ps=case.alpha_ps, beta_ps=case.beta_ps,
                      n_sat=case.n_sat, capacity_factor=case.capacity_factor,
                      bw_bytes_per_us=case.bw_bytes_per_us, dtype=case.dtype,
                      dedup_wire=case.dedup_wire or case.predispatch, predispatch=case.predispatch,
                      fuse_gate_predictor=case.fuse_gate_predictor)
    rt = ProbeRuntime(cfg)
    if case.ep_emulation:
        from paper_2602_00509_b200._lib import OPT_EP_EMULATION
        rt.set_option(OPT_EP_EMULATION, 1)
    if not case.pair_gemm:
        from paper_2602_00509_b200._lib import OPT_PAIR_GEMM
        rt.set_option(OPT_PAIR_GEMM, 0)
    if case.fused_epi_topk:
        from paper_2602_00509_b200._lib import OPT_FUSED_EPILOGUE_TOPK
        rt.set_option(OPT_FUSED_EPILOGUE_TOPK, 1)
    dev = "cuda"
    if case.gen == "natural":
        L0 = pi.natural_layer_inputs(sh, case.step, 0, device=dev)
        L1 = pi.natural_layer_inputs(sh, case.step, 1, device=dev)
        W, b = map(list, zip(*[pi.natural_router(sh, p, case.step, case.zipf_s, device=dev) for p in (0, 1)]))
    else:
        L0 = pi.layer_inputs(sh, case.step, 0, case.zipf_s, device=dev)
        L1 = pi.layer_inputs(sh, case.step, 1, case.zipf_s, device=dev)
        W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
        b = [None, None]
        if case.bias:
            b = [torch.from_numpy((np.arange(E) % 4 - 1.5).astype(np.float32) / 64).to(dev) for _ in (0, 1)]
    w13 = [None, None]
    w2 = [None, None]
    for p in (0, 1):
        w13[p], w2[p] = pi.expert_weights(sh, p, device=dev, dtype=cfg.torch_dtype)
    if case.residual_kind == "relabel":
        r1, r2 = pi.predictor_residual_relabel(sh, 1, device=dev)
    else:
        r1, r2 = pi.predictor_residual(sh, 1, zero=not case.residual, device=dev)
    if not case.residual:
        r1 = r2 = None
    if case.dtype == "fp32":   # routing inputs keep their (exact) generator values, stored as fp32
        L0.x, L1.x = L0.x.float(), L1.x.float()
        W = [w.float() for w in W]
        if r1 is not None:
            r1, r2 = r1.float(), r2.float()
    odt = torch.float32 if case.out_fp32 else torch.bfloat16
    out = [torch.empty(G, T, H, dtype=odt, device=dev) for _ in (0, 1)]
    ids = [torch.empty(G, T, k, dtype=torch.int32, device=dev) for _ in (0, 1)]
    gw = [torch.empty(G, T, k, dtype=torch.float32, device=dev) for _ in (0, 1)]
    pc = torch.empty(G, E, dtype=torch.int32, device=dev)
    plog = torch.empty(G, T, E, dtype=torch.float32, device=dev)
    reps = torch.empty(G, 3, dtype=torch.int32, device=dev)
    quota = torch.empty(G, E, G, dtype=torch.int32, device=dev)
    stats = torch.empty(8, dtype=torch.int64, device=dev)
    win = torch.full((G,), case.window_ns, dtype=torch.int64, device=dev)
    res = {}
    if case.fuse_gate_predictor:        # layer 0's gate GEMM also computes stage 1 of layer 1's predictor
        rt.predict_prepare(1, W[1], r1)
    rt.forward(0, L0.x, W[0], b[0], w13[0], w2[0], out[0], use_plan=False, topk_ids=ids[0], topk_w=gw[0])
    if os.environ.get("PROBE_TEST_SYNC_L0"):      # debugging aid: serialise layer 0 before the aux track
        torch.cuda.synchronize()
    lay0 = debug(rt, cfg, T, L0.x)
    # the product path both times: once also returning the logits k_select ranks, once as the bench runs it
    pc_logits = torch.empty(G, E, dtype=torch.int32, device=dev)
    rt.predict(1, L0.x, W[1], b[1], r1, r2, pred_counts=pc_logits, pred_logits=plog)
    rt.predict(1, L0.x, W[1], b[1], r1, r2, pred_counts=pc)
    rt.plan(1, win, replicas=reps, quota=quota, stats=stats)
    rt.prefetch(1, w13[1], w2[1], phase=0)
    rt.forward(1, L1.x, W[1], b[1], w13[1], w2[1], out[1], use_plan=True, topk_ids=ids[1], topk_w=gw[1])
    lay1 = debug(rt, cfg, T, L1.x)
    res["flags"] = rt.flags()
    rt.check()
    torch.cuda.synchronize()
    res.update(out=[o.float().cpu().numpy() for o in out], ids=[i.cpu().numpy() for i in ids],
               g=[g.cpu().numpy() for g in gw], pred_counts=pc.cpu().numpy(), pred_logits=plog.cpu().numpy(),
               pred_counts_logits=pc_logits.cpu().numpy(),
               replicas=reps.cpu().numpy(), quota=quota.cpu().numpy(), stats=stats.cpu().numpy(),
               layout=[lay0, lay1])
    # replica slots (bank 1 for layer 1) must hold the home expert's weights bit-exactly
    slots = []
    for r in range(G):
        sw13, sw2 = rt.replica_slots(r)
        for q in range(3):
            e = int(res["replicas"][r, q])
            if e >= 0:
                slots.append(bool(torch.equal(sw13[3 + q].view(torch.uint8), w13[1][e].view(torch.uint8)) and
                                  torch.equal(sw2[3 + q].view(torch.uint8), w2[1][e].view(torch.uint8))))
    res["slots_ok"] = slots
    inputs = dict(L0=L0, L1=L1, W=W, b=b, w13=w13, w2=w2, r1=r1, r2=r2)
    rt.close()
    return res, inputs


def debug(rt, cfg, T=None, x=None):
    G, E, k = cfg.G, cfg.E, cfg.k
    T = cfg.T if T is None else T
    S = E // G + 3
    counts = torch.empty(G, E, dtype=torch.int32, device="cuda")
    split = torch.empty(G, E, G, dtype=torch.int32, device="cuda")
    route = torch.empty(G, T, k, 2, dtype=torch.int32, device="cuda")
    rows = torch.empty(G, S, dtype=torch.int32, device="cuda")
    reps = torch.empty(G, 3, dtype=torch.int32, device="cuda")
    rt.debug_layout(counts, split, route, rows, reps)
    torch.cuda.synchronize()
    out = dict(counts=counts.cpu().numpy(), split_cum=split.cpu().numpy(), route=route.cpu().numpy(),
               group_rows=rows.cpu().numpy(), replicas=reps.cpu().numpy())
    if x is not None:
        out["recv_ok"] = recv_rows_match(rt, cfg, x, route)
    return out


def recv_rows_match(rt, cfg, x, route):
    """Dispatch payload pin (a6): every routed (token, slot) row of every destination's receive
    buffer equals the source's x row bit for bit (after the dedup expansion when enabled)."""
    from paper_2602_00509_b200 import _lib
    G, H, cap = cfg.G, cfg.H, cfg.recv_capacity
    recv = torch.stack([rt.sym_view(_lib.BUF_RECV, r, x.dtype, (cap, H)) for r in range(G)])
    dd, rr = route[..., 0].long(), route[..., 1].long()
    valid = rr >= 0
    ok = True
    for s in range(x.shape[0]):                      # per source rank (bounded memory at full size)
        got = recv[dd[s].clamp(min=0), rr[s].clamp(min=0)]            # [T, k, H]
        same = (got == x[s][:, None, :]) | (got.isnan() & x[s][:, None, :].isnan())
        ok &= bool((same | ~valid[s][..., None]).all())
    return ok


def sampled_tokens(case: CaseCfg):
    if case.sample_tokens <= 0:
        return None
    sh = case.shape
    r = np.random.default_rng(77)
    out = []
    for s in range(sh.G):
        t = np.sort(r.choice(sh.T, size=min(case.sample_tokens, sh.T), replace=False))
        t[-1] = sh.T - 1                     # always include the ragged tail token
        out.append(sorted(set(int(v) for v in t)))
    return out


def run_oracle(case: CaseCfg, inputs, tokens=None):
    sh = case.shape
    tokens = sampled_tokens(case) if tokens is None else tokens
    G, E, k = sh.G, sh.E, sh.k
    W = [f64(w) for w in inputs["W"]]
    b = [None if v is None else v.double().cpu().numpy() for v in inputs["b"]]
    xs0 = [f64(inputs["L0"].x[r]) for r in range(G)]
    xs1 = [f64(inputs["L1"].x[r]) for r in range(G)]
    W13 = [LazyExperts(inputs["w13"][p]) for p in (0, 1)]
    W2 = [LazyExperts(inputs["w2"][p]) for p in (0, 1)]
    r1 = None if inputs["r1"] is None else f64(inputs["r1"])
    r2 = None if inputs["r2"] is None else f64(inputs["r2"])
    ref0 = O.layer_reference(xs0, W[0], b[0], k, None, G, E, W13[0], W2[0], tokens)
    nhat, plog, nhat_prior = [], [], []
    for r in range(G):
        l, _ = O.predictor_logits(xs0[r], W[1], b[1], r1, r2)
        plog.append(l)
        nhat.append(np.bincount(O.topk_ids(l, k).reshape(-1), minlength=E))
        lp, _ = O.predictor_logits(xs0[r], W[1], b[1], None, None)
        nhat_prior.append(np.bincount(O.topk_ids(lp, k).reshape(-1), minlength=E))
    nhat = np.stack(nhat)
    pcfg = O.PlannerConfig(G=G, E=E, replica_budget=case.replica_budget, kmax=16, alpha_ps=case.alpha_ps,
                           beta_ps=case.beta_ps, n_sat=case.n_sat, bw_bytes_per_us=case.bw_bytes_per_us,
                           expert_bytes=3 * sh.H * sh.F * case.es)
    plan = O.plan_greedy(nhat, [case.window_ns] * G, pcfg)
    ref1 = O.layer_reference(xs1, W[1], b[1], k, plan, G, E, W13[1], W2[1], tokens)
    return dict(ref=[ref0, ref1], nhat=nhat, plan=plan, pred_logits=np.stack(plog), tokens=tokens,
                residual_changes_nhat=not np.array_equal(nhat, np.stack(nhat_prior)))


def group_rows_oracle(lay: O.Layout, G, E):
    S = E // G + 3
    out = np.zeros((G, S), dtype=np.int64)
    for r in range(G):
        sz = lay.group_sizes[r]
        out[r, :len(sz)] = sz
    return out


def half_ulp_bf16(v):
    """Half a bf16 ulp at |v| (8 significant bits): 2^(floor(log2|v|) - 8); 0 at v = 0."""
    v = np.asarray(v, dtype=np.float64)
    m, e = np.frexp(v)                      # v = m·2^e, m in [0.5, 1)  ⇒ floor(log2 v) = e - 1
    return np.where(v > 0, np.ldexp(1.0, e - 1 - 8), 0.0)


def compare(case: CaseCfg, gpu, orc, tol: float = 2e-2):
    """Bit-exact: ids, counts, predicted counts, plan, split, route, group sizes, replica bytes.
    Tolerance: gate weights (1e-6 abs), predictor logits (1e-5 rel), outputs (tol · RMS)."""
    sh = case.shape
    G, E, k = sh.G, sh.E, sh.k
    report = {}
    for L in (0, 1):
        ref = orc["ref"][L]
        for r in range(G):
            assert np.array_equal(gpu["ids"][L][r], ref["ids"][r]), f"ids L{L} r{r}"
            assert np.abs(gpu["g"][L][r] - ref["g"][r]).max() < 1e-6, f"gate weights L{L} r{r}"
        lay = gpu["layout"][L]
        assert np.array_equal(lay["counts"], ref["n"]), f"counts L{L}"
        assert np.array_equal(lay["split_cum"], np.cumsum(ref["split"], axis=2)), f"split L{L}"
        for r in range(G):
            assert np.array_equal(lay["route"][r, :, :, 0], ref["layout"].dest[r]), f"route dest L{L} r{r}"
            assert np.array_equal(lay["route"][r, :, :, 1], ref["layout"].row[r]), f"route row L{L} r{r}"
        assert np.array_equal(lay["group_rows"], group_rows_oracle(ref["layout"], G, E)), f"group rows L{L}"
        if "recv_ok" in lay:
            assert lay["recv_ok"], f"receive rows differ from the dispatched x rows L{L}"
        errs, excess = [], []
        rms = np.sqrt(np.mean(np.concatenate([o.reshape(-1) for o in ref["out"]]) ** 2))
        toks = orc.get("tokens")
        for r in range(G):
            got = gpu["out"][L][r] if toks is None else gpu["out"][L][r][toks[r]]
            err = np.abs(got - ref["out"][r])
            errs.append(err.max())
            # bf16 output = the fp32 result rounded to bf16: each element may additionally be off by
            # half a bf16 ulp of its value (2^(floor(log2|v|) - 8)); the 2e-2·RMS bound applies to the rest
            rnd = 0.0 if case.out_fp32 else half_ulp_bf16(np.maximum(np.abs(got), np.abs(ref["out"][r])))
            excess.append((err - rnd).max())
        report[f"out_err_L{L}"] = float(max(errs) / rms)
        if not case.out_fp32:
            report[f"out_err_beyond_bf16_rounding_L{L}"] = float(max(excess) / rms)
        assert max(excess) <= tol * rms, f"output L{L}: max err {max(excess)} > {tol} * RMS {rms}"
    assert np.array_equal(gpu["pred_counts"], orc["nhat"]), "predicted counts"
    assert np.array_equal(gpu["pred_counts_logits"], orc["nhat"]), "predicted counts (call returning logits)"
    pl = orc["pred_logits"]
    report["pred_logit_err"] = float(np.abs(gpu["pred_logits"] - pl).max())
    assert report["pred_logit_err"] <= 1e-5 * max(1.0, np.abs(pl).max()), "predictor logits"
    plan = orc["plan"]
    exp_reps = np.full((G, 3), -1)
    for r in range(G):
        exp_reps[r, :len(plan.replicas[r])] = plan.replicas[r]
    assert np.array_equal(gpu["replicas"], exp_reps), f"replicas {gpu['replicas'].tolist()} vs {exp_reps.tolist()}"
    assert np.array_equal(gpu["quota"], plan.quota), "quota"
    assert gpu["stats"][0] == plan.iterations and gpu["stats"][2] == plan.maxL_before \
        and gpu["stats"][3] == plan.maxL_after, f"plan stats {gpu['stats']}"
    assert all(gpu["slots_ok"]), "replica slot bytes differ from home expert weights"
    report["replicas"] = int((exp_reps >= 0).sum())
    report["residual_changes_nhat"] = bool(orc["residual_changes_nhat"])
    if case.predispatch:
        report["predispatch_hits"], report["predispatch_misses"] = gpu["flags"][5], gpu["flags"][6]
    report["iterations"] = plan.iterations
    return report

"""GPU parity of the whole PROBE layer (all §8(a) rows) against the fp64 oracle.

Single-GPU emulation of G logical EP ranks (every peer pointer maps into this
device).  Bit-exact: routing ids, actual/predicted counts, plan (replicas,
quota, stats), materialized split, dispatch route (dest, row), group sizes,
replica slot bytes.  Tolerance: outputs within 2e-2·RMS (bf16 tensor-core path
with fp32 output, north_star), gate weights 1e-6.
"""
import numpy as np
import pytest
import torch

import oracle as O
import probe_inputs as pi
from layer_harness import CaseCfg, compare, f64, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = {
    "C0": CaseCfg(pi.C0, zipf_s=1.5),
    "C0-comm-nsat": CaseCfg(pi.C0, zipf_s=1.2, alpha_ps=3, beta_ps=2, n_sat=4, step=1),
    "mid-ragged": CaseCfg(pi.C0.with_(name="mid", E=32, k=4, H=512, F=256, T=200, G=4), zipf_s=1.2, bias=True),
    "G8-E64": CaseCfg(pi.C0.with_(name="g8", E=64, k=8, H=512, F=384, T=160, G=8), zipf_s=1.0, alpha_ps=5,
                      beta_ps=1, n_sat=16),
    "G1": CaseCfg(pi.C0.with_(name="g1", E=16, k=4, H=256, F=256, T=300, G=1), zipf_s=1.0),
    "bf16-out": CaseCfg(pi.C0.with_(name="bf", E=16, k=4, H=256, F=256, T=96, G=2), out_fp32=False),
    "no-residual": CaseCfg(pi.C0.with_(name="nr", E=16, k=2, H=256, F=128, T=64, G=2), residual=False),
    "budget0": CaseCfg(pi.C0, replica_budget=0),
    "fused-epilogue-topk": CaseCfg(pi.C0.with_(name="fe", E=64, k=8, H=512, F=256, T=200, G=4), zipf_s=1.3,
                                  fused_epi_topk=True, bias=True),
    "one-cta-gemm": CaseCfg(pi.C0.with_(name="pg", E=32, k=4, H=512, F=384, T=333, G=4), zipf_s=1.3,
                            pair_gemm=False),
    "one-cta-gemm-ep-emulation": CaseCfg(pi.C0.with_(name="pge", E=64, k=8, H=512, F=256, T=256, G=8), zipf_s=1.2,
                                         pair_gemm=False, ep_emulation=True),
    "ep-emulation": CaseCfg(pi.C0.with_(name="epem", E=64, k=8, H=512, F=384, T=300, G=8), zipf_s=1.2,
                            ep_emulation=True),
    # CTA-pair expert GEMMs (chosen when T·k·G/E ≥ 256 rows per local expert)
    "pair-gemm": CaseCfg(pi.C0.with_(name="pgl", E=16, k=4, H=256, F=256, T=700, G=4), zipf_s=1.3),
    "pair-gemm-ep-emulation": CaseCfg(pi.C0.with_(name="pgle", E=16, k=4, H=256, F=384, T=600, G=4), zipf_s=1.2,
                                      ep_emulation=True),
    # degenerate top-k: k = 1, k = E (every expert chosen by every token), k = 9 > 8 (unfused select kernel; the exact-bf16 encoding caps k near 9)
    "k1": CaseCfg(pi.C0.with_(name="k1", E=8, k=1, H=256, F=256, T=130, G=2), zipf_s=1.5),
    "k-eq-E": CaseCfg(pi.C0.with_(name="kE", E=8, k=8, H=256, F=128, T=70, G=2), zipf_s=1.0),
    "k9-unfused-select": CaseCfg(pi.C0.with_(name="k9b", E=32, k=9, H=256, F=128, T=100, G=2), zipf_s=1.2),
    # H, F not multiples of the 256-column tile: ragged N in GEMM1 (2F) and GEMM2 (H), ragged K
    "ragged-HF": CaseCfg(pi.C0.with_(name="rhf", E=16, k=4, H=320, F=320, T=64, G=2), zipf_s=1.3),
    # ...with groups of >= 32 rows, so the last N tile mixes TMA-stored chunks with chunks past
    # N (the fp16-Y staging-slot reuse bug: columns 2848..2879 of C2's Y were overwritten)
    "ragged-HF-tma": CaseCfg(pi.C0.with_(name="rhft", E=16, k=4, H=320, F=320, T=600, G=2), zipf_s=1.0),
    "ragged-HF-tma-one-cta": CaseCfg(pi.C0.with_(name="rhfo", E=16, k=4, H=320, F=320, T=600, G=2), zipf_s=1.0,
                                     pair_gemm=False),
    "C2-dims-static": CaseCfg(pi.C0.with_(name="c2s", E=16, k=4, H=2880, F=2880, T=64, G=2), zipf_s=1.3,
                              replica_budget=0),
    "C2-dims": CaseCfg(pi.C0.with_(name="c2d", E=16, k=4, H=2880, F=2880, T=64, G=2), zipf_s=1.3),
    # natural generator: dyadic x / router, negative and dense logits, exact ties
    # from duplicated router rows, Zipf skew through a dyadic bias
    "natural-C0": CaseCfg(pi.C0, zipf_s=1.2, gen="natural", residual=False),
    "natural-mid": CaseCfg(pi.C0.with_(name="natm", E=64, k=8, H=512, F=256, T=300, G=4), zipf_s=1.2,
                           gen="natural", residual=False),
    "natural-mid-bf16-out": CaseCfg(pi.C0.with_(name="natb", E=32, k=4, H=768, F=256, T=257, G=4), zipf_s=1.0,
                                    gen="natural", residual=False, out_fp32=False),
    # a predictor residual that changes n̂ (exact relabelling), through the product path
    "relabel-residual-C0": CaseCfg(pi.C0, zipf_s=1.2, residual_kind="relabel"),
    "relabel-residual-mid": CaseCfg(pi.C0.with_(name="rl", E=32, k=4, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                    residual_kind="relabel", bias=True),
    "relabel-residual-epilogue-topk": CaseCfg(pi.C0.with_(name="rle", E=64, k=8, H=512, F=256, T=200, G=4),
                                              zipf_s=1.3, residual_kind="relabel", fused_epi_topk=True),
    # dedup wire (§8(a) a6/a8): one row per unique (token, dest) + receiver expansion; expert-side
    # fp32 partials per (token, dest) pushed to the source, summed in ascending dest order (R25)
    "dedup-C0": CaseCfg(pi.C0, zipf_s=1.5, dedup_wire=True),
    "dedup-G8-E64": CaseCfg(pi.C0.with_(name="dg8", E=64, k=8, H=512, F=384, T=160, G=8), zipf_s=1.0, alpha_ps=5,
                            beta_ps=1, n_sat=16, dedup_wire=True),
    "dedup-pair-gemm-bias": CaseCfg(pi.C0.with_(name="dpg", E=16, k=4, H=256, F=256, T=700, G=4), zipf_s=1.3,
                                    bias=True, dedup_wire=True),
    "dedup-bf16-out": CaseCfg(pi.C0.with_(name="dbf", E=16, k=4, H=256, F=256, T=96, G=2), out_fp32=False,
                              dedup_wire=True),
    "dedup-ragged-HF-ep-emulation": CaseCfg(pi.C0.with_(name="drh", E=32, k=8, H=320, F=320, T=300, G=4),
                                            zipf_s=1.2, ep_emulation=True, dedup_wire=True),
    "dedup-k-eq-E": CaseCfg(pi.C0.with_(name="dkE", E=8, k=8, H=256, F=128, T=70, G=2), zipf_s=1.0,
                            dedup_wire=True),
    "dedup-natural": CaseCfg(pi.C0.with_(name="dnat", E=64, k=8, H=512, F=256, T=300, G=4), zipf_s=1.2,
                             gen="natural", residual=False, dedup_wire=True),
    # NEXT-4 predictive pre-dispatch: layer 1 rows pushed to the predicted experts' home ranks
    # during its gate; only missed (token, dest) pairs ship after the gate; hits expand from PRE
    "predispatch-C0": CaseCfg(pi.C0, zipf_s=1.5, predispatch=True),
    "predispatch-G8-E64": CaseCfg(pi.C0.with_(name="pd8", E=64, k=8, H=512, F=384, T=160, G=8), zipf_s=1.0,
                                  alpha_ps=5, beta_ps=1, n_sat=16, predispatch=True),
    "predispatch-relabel-ragged": CaseCfg(pi.C0.with_(name="pdr", E=32, k=4, H=320, F=320, T=301, G=4), zipf_s=1.2,
                                          residual_kind="relabel", bias=True, predispatch=True),
    "predispatch-T-below-capacity": CaseCfg(pi.C0.with_(name="pdt", E=16, k=4, H=256, F=256, T=77, G=4),
                                            zipf_s=1.3, max_tokens=300, predispatch=True),
    # predictor residual width h = H/4 >= 256: Ŵ1·x on CTA pairs (PROBE_OPT_PRED_PAIR), ragged T
    "predictor-pair-gemm": CaseCfg(pi.C0.with_(name="ppg", E=32, k=4, H=1024, F=256, T=301, G=4), zipf_s=1.2,
                                   bias=True),
    "predictor-pair-gemm-relabel": CaseCfg(pi.C0.with_(name="ppr", E=64, k=8, H=1536, F=256, T=200, G=4),
                                           zipf_s=1.2, residual_kind="relabel"),
    # fused gate + predictor stage 1 (probe_config.fuse_gate_predictor): layer 0's gate GEMM over
    # [W_0 ; W_1 ; Ŵ1] (row-chunk interleaved groups, split fp32 epilogue, TMA bf16 activation),
    # then layer 1's predictor runs only Ŵ2·a (out-of-place accumulate) + select
    "gate-fused-predictor": CaseCfg(pi.C0.with_(name="gfp", E=32, k=4, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                    fuse_gate_predictor=True),
    "gate-fused-predictor-relabel-bias": CaseCfg(pi.C0.with_(name="gfr", E=64, k=8, H=1536, F=256, T=200, G=4),
                                                 zipf_s=1.2, residual_kind="relabel", bias=True,
                                                 fuse_gate_predictor=True),
    "gate-fused-predictor-one-cta": CaseCfg(pi.C0.with_(name="gf1", E=32, k=4, H=256, F=256, T=50, G=2),
                                            zipf_s=1.3, fuse_gate_predictor=True),
    "gate-fused-prior-only": CaseCfg(pi.C0.with_(name="gfn", E=32, k=4, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                     residual=False, fuse_gate_predictor=True),
    "gate-fused-ragged-h": CaseCfg(pi.C0.with_(name="gfh", E=32, k=4, H=320, F=320, T=300, G=4), zipf_s=1.3,
                                   bias=True, fuse_gate_predictor=True),    # h = 80: manual bf16 stores
    "gate-fused-ep-emulation": CaseCfg(pi.C0.with_(name="gfem", E=64, k=8, H=512, F=384, T=300, G=8), zipf_s=1.2,
                                       ep_emulation=True, fuse_gate_predictor=True),   # the bench's emulated line
    "gate-fused-E256": CaseCfg(pi.C0.with_(name="gfe", E=256, k=8, H=1024, F=128, T=64, G=8), zipf_s=1.0,
                               residual_kind="relabel", fuse_gate_predictor=True),
    # the dedup-natural draw ("dnat") again, with pre-dispatch and the fused gate on top; on
    # another draw of this shape ("gfpd") the bf16 activation rounding ALONE (CPU emulation:
    # round_bf16(SwiGLU) then fp16 Y) reaches 2.2e-2·RMS, above north_star's bound
    "gate-fused-natural-predispatch": CaseCfg(pi.C0.with_(name="dnat", E=64, k=8, H=512, F=256, T=300, G=4),
                                              zipf_s=1.2, gen="natural", residual=False, predispatch=True,
                                              fuse_gate_predictor=True),
    "predispatch-natural": CaseCfg(pi.C0.with_(name="dnat", E=64, k=8, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                   gen="natural", residual=False, predispatch=True),
    # the layer call runs with T below the context's max_tokens (workspaces sized for 4x more)
    "T-below-capacity": CaseCfg(pi.C0.with_(name="tbc", E=16, k=4, H=256, F=256, T=77, G=4), zipf_s=1.3,
                                max_tokens=300),
}


@pytest.mark.parametrize("name", list(CASES))
def test_layer_parity(name):
    case = CASES[name]
    gpu, inputs = run_gpu(case)
    orc = run_oracle(case, inputs)
    rep = compare(case, gpu, orc, tol=2e-2)
    print(name, rep)
    if name == "budget0":
        assert rep["replicas"] == 0
    if case.residual_kind == "relabel":
        assert rep["residual_changes_nhat"]
    if case.predispatch:
        assert rep["predispatch_hits"] > 0 and rep["predispatch_hits"] + rep["predispatch_misses"] > 0


def test_static_ep_identity_and_plan_independence():
    """With replication disabled the layer is plain static EP; with a plan the output is
    the same function (semantic equivalence) up to fp32 summation order."""
    case = CASES["C0"]
    gpu, inputs = run_gpu(case)
    sh = case.shape
    # static EP layout: every (token, slot) goes to its expert's home rank
    lay0 = gpu["layout"][0]
    for r in range(sh.G):
        assert np.array_equal(lay0["route"][r, :, :, 0], gpu["ids"][0][r] // (sh.E // sh.G))
    assert gpu["replicas"].max() >= 0, "expected the planner to replicate under s=1.5"


def test_fp16_y_range_is_checked():
    """D2: Y is stored in fp16; an expert output beyond ±65504 must not pass silently —
    probe_check reports PROBE_ESHAPE (device error bit set by the GEMM2 epilogue)."""
    import torch
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    from paper_2602_00509_b200._lib import ProbeError
    sh = pi.C0
    rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h))
    li = pi.layer_inputs(sh, 0, 0, 1.2, device="cuda")
    W = pi.router_weight(sh, 0, device="cuda")
    w13, w2 = pi.expert_weights(sh, 0, device="cuda")
    out = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    rt.forward(0, li.x, W, None, w13, w2, out)
    rt.check()                                        # in range: no error
    rt.forward(0, li.x, W, None, w13, (w2.float() * 2.0 ** 26).to(torch.bfloat16), out)   # |y| ≈ 1.7e6
    with pytest.raises(ProbeError, match="65504"):
        rt.check()
    rt.close()


# fp32 parity path (probe_config.dtype = PROBE_FP32): north_star's fp32 bound, 1e-5·RMS.  fp32
# expert weights (full fp32 draws, not bf16 values), SIMT fp32 GEMMs, fp32 Y and combine; routing,
# plan and layout must still be bit-exact.  Cases span several 64×64 SIMT tiles with ragged tails.
FP32_CASES = {
    "fp32-C0": CaseCfg(pi.C0, zipf_s=1.5, dtype="fp32"),
    "fp32-mid-ragged": CaseCfg(pi.C0.with_(name="mid32", E=32, k=4, H=512, F=256, T=200, G=4), zipf_s=1.2,
                               bias=True, dtype="fp32"),
    "fp32-G8-E64": CaseCfg(pi.C0.with_(name="g832", E=64, k=8, H=512, F=384, T=160, G=8), zipf_s=1.0,
                           alpha_ps=5, beta_ps=1, n_sat=16, dtype="fp32"),
    "fp32-G1": CaseCfg(pi.C0.with_(name="g132", E=16, k=4, H=256, F=320, T=300, G=1), zipf_s=1.0, dtype="fp32"),
    "fp32-no-residual-budget0": CaseCfg(pi.C0.with_(name="nr32", E=16, k=2, H=256, F=128, T=64, G=2),
                                        residual=False, replica_budget=0, dtype="fp32"),
    "fp32-dedup-G8": CaseCfg(pi.C0.with_(name="d832", E=64, k=8, H=512, F=256, T=160, G=8), zipf_s=1.0,
                             dtype="fp32", dedup_wire=True),
    # the natural-generator draw whose bf16 activation rounding alone exceeds 2e-2·RMS: the fp32
    # path on it (per-slot and dedup wire) is within 1e-5·RMS, so the bf16 excess is the
    # activation's rounding point, not the routing, layout, wire or combine
    "fp32-natural-gfpd": CaseCfg(pi.C0.with_(name="gfpd", E=64, k=8, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                 gen="natural", residual=False, dtype="fp32"),
    "fp32-natural-gfpd-dedup": CaseCfg(pi.C0.with_(name="gfpd", E=64, k=8, H=512, F=256, T=300, G=4), zipf_s=1.2,
                                       gen="natural", residual=False, dtype="fp32", dedup_wire=True),
}


@pytest.mark.parametrize("name", list(FP32_CASES))
def test_layer_parity_fp32(name):
    case = FP32_CASES[name]
    gpu, inputs = run_gpu(case)
    orc = run_oracle(case, inputs)
    rep = compare(case, gpu, orc, tol=1e-5)
    print(name, rep)


def test_boundary_errors():
    """Host-checkable errors (include/probe.h): T outside [1, max_tokens] → PROBE_ECAPACITY,
    use_plan without probe_plan/probe_prefetch for that layer → PROBE_ESTATE, null pointers →
    PROBE_EINVAL; the context stays usable after each refused call."""
    import torch
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    from paper_2602_00509_b200._lib import ProbeError
    sh = pi.C0
    rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h))
    li = pi.layer_inputs(sh, 0, 0, 1.2, device="cuda")
    W = pi.router_weight(sh, 0, device="cuda")
    w13, w2 = pi.expert_weights(sh, 0, device="cuda")
    out = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    big = torch.zeros(sh.G, sh.T + 1, sh.H, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ProbeError, match="CAPACITY"):
        rt.forward(0, big, W, None, w13, w2, out)
    from paper_2602_00509_b200._lib import STATUS
    from paper_2602_00509_b200.runtime import _ptr
    st = rt.lib.probe_moe_forward(rt.ctx, 0, _ptr(li.x), 0, _ptr(W), None, _ptr(w13), _ptr(w2), 0, _ptr(out), 1,
                                  None, None, None)                       # T = 0, valid pointers
    assert STATUS[st] == "PROBE_ECAPACITY"
    with pytest.raises(ProbeError, match="STATE"):
        rt.forward(3, li.x, W, None, w13, w2, out, use_plan=True)
    with pytest.raises(ProbeError, match="INVAL"):
        rt.forward(0, li.x, W, None, w13, None, out)
    with pytest.raises(ProbeError, match="STATE"):   # fuse_gate_predictor is off in this config
        rt.predict_prepare(1, W)
    rt.forward(0, li.x, W, None, w13, w2, out)      # still usable
    rt.check()
    assert torch.isfinite(out).all()
    rt.close()


def test_fused_gate_prediction_falls_back_on_other_operands():
    """probe_predict_prepare arms the gate of ONE forward; probe_predict then reuses its stage 1
    only for exactly the armed operands.  A predict with another x (or weights) recomputes stage 1
    itself, so n̂ never depends on the arming."""
    import torch
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    sh = pi.C0.with_(name="gff", E=32, k=4, H=512, F=256, T=128, G=4)
    rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h,
                                  fuse_gate_predictor=True))
    L0 = pi.layer_inputs(sh, 0, 0, 1.2, device="cuda")
    L1 = pi.layer_inputs(sh, 0, 1, 1.2, device="cuda")
    W = [pi.router_weight(sh, p, device="cuda") for p in (0, 1)]
    w13, w2 = pi.expert_weights(sh, 0, device="cuda")
    r1, r2 = pi.predictor_residual_relabel(sh, 1, device="cuda")
    out = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    pcs = [torch.empty(sh.G, sh.E, dtype=torch.int32, device="cuda") for _ in range(3)]
    rt.predict_prepare(1, W[1], r1)
    rt.forward(0, L0.x, W[0], None, w13, w2, out)
    rt.predict(1, L0.x, W[1], None, r1, r2, pred_counts=pcs[0])     # reuses the fused stage 1
    rt.predict(1, L1.x, W[1], None, r1, r2, pred_counts=pcs[1])     # other x: recomputed
    rt.predict(1, L0.x, W[1], None, r1, r2, pred_counts=pcs[2])     # back to the armed x: reused again
    rt.check()
    torch.cuda.synchronize()
    x0 = [f64(L0.x[r]) for r in range(sh.G)]
    x1 = [f64(L1.x[r]) for r in range(sh.G)]
    W1, a, b = f64(W[1]), f64(r1), f64(r2)
    exp0 = np.stack([O.predict_counts(x0[r], W1, None, a, b, sh.k)[0] for r in range(sh.G)])
    exp1 = np.stack([O.predict_counts(x1[r], W1, None, a, b, sh.k)[0] for r in range(sh.G)])
    assert np.array_equal(pcs[0].cpu().numpy(), exp0)
    assert np.array_equal(pcs[1].cpu().numpy(), exp1)
    assert np.array_equal(pcs[2].cpu().numpy(), exp0)
    assert not np.array_equal(exp0, exp1)
    rt.close()

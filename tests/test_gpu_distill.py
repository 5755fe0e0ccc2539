"""GPU: online distillation of the predictor residual (NEXT-1, R33-R37) through
the C-ABI (probe_distill_grad / probe_distill_apply) against the fp64 oracle.

Tolerances: teacher logits 1e-5·RMS (bf16 operands, fp32 accumulation);
student logits 2e-3·RMS (the bf16 activation can round the other way where the GPU's fp32
SiLU and the oracle's fp64 SiLU straddle a bf16 midpoint); summed CE 1e-3 relative; the
gradients ELEMENT-WISE: max_ij |∇_gpu − ∇_oracle| <= 2e-2 · RMS(∇_oracle), the layer-output
criterion.  Derivation: each gradient element is a token sum Σ_t u_t v_t whose operands
(q − p, g_z) are rounded to bf16 (R35, relative 2^-9 each); the rounding errors are
independent across t, so the error is ≈ 2^-9·sqrt(Σ_t (u_t v_t)^2), while the element
itself is a sum of mixed-sign terms of the same size (RMS ≈ sqrt(Σ (u v)^2)): error/RMS ≈
2^-9 per element, ≈ 1e-2 at the maximum over 10^5 elements; fidelity hit counts
bit-exact, decided on the GPU's own fp32 logits on both sides (③).
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import probe_inputs as pi

pytestmark = pytest.mark.gpu

CASES = {
    "C0": (pi.C0, 64),
    "mid-ragged": (pi.C0.with_(name="dmid", E=32, k=4, H=512, T=200, G=2, h=128), 200),
    "E256-k8": (pi.C0.with_(name="d256", E=256, k=8, H=1024, T=150, G=1, h=256), 150),
    "h-tail": (pi.C0.with_(name="dht", E=64, k=6, H=256, T=77, G=4, h=40), 77),
    # N = 3000 tokens: both token contractions run split-K (5 K-splits + ordered reduction)
    "split-k": (pi.C0.with_(name="dsk", E=32, k=4, H=512, T=1500, G=2, h=128), 1500),
}


def _setup(sh, seed, w2_scale=0.5, zero_w2=False, same_x=False):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    task = pi.distill_task(sh, seed, device="cuda")
    rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=64, T=sh.T, h=sh.h))
    g = pi.torch_gen(sh.name, seed, "distill-test")
    w1 = (torch.randn(sh.h, sh.H, generator=g) / math.sqrt(sh.H)).to(torch.bfloat16).cuda()
    w2 = (torch.randn(sh.E, sh.h, generator=g) * w2_scale / math.sqrt(sh.h)).to(torch.bfloat16).cuda()
    if zero_w2:
        w2.zero_()
    b = (torch.randn(sh.E, generator=g) * 0.1).cuda()
    xn = task.x if same_x else task.x_next
    return rt, task.x, xn, task.W, b, w1, w2


def _np(t):
    return pi.bf16_to_numpy_f64(t) if t.dtype == torch.bfloat16 else t.double().cpu().numpy()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", list(CASES))
def test_distill_grad_parity(name):
    sh, T = CASES[name]
    rt, x, xn, W, b, w1, w2 = _setup(sh, 0)
    N = sh.G * T
    g1 = torch.empty(sh.h, sh.H, device="cuda")
    g2 = torch.empty(sh.E, sh.h, device="cuda")
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    sl = torch.empty(N, sh.E, device="cuda")
    tl = torch.empty(N, sh.E, device="cuda")
    rt.distill_grad(x, xn, W, b, w1, w2, g1, g2, stats, sl, tl)
    torch.cuda.synchronize()
    rt.check()
    X, XN, Wn, bn = _np(x).reshape(N, sh.H), _np(xn).reshape(N, sh.H), _np(W), _np(b)
    loss, o1, o2, f = O.distill_grads(X, XN, Wn, bn, _np(w1), _np(w2))
    s = stats.cpu().numpy()
    t_gpu = tl.double().cpu().numpy() + bn
    l_gpu = sl.double().cpu().numpy() + bn
    assert np.abs(t_gpu - f["t"]).max() <= 1e-5 * np.sqrt((f["t"] ** 2).mean()), "teacher logits"
    assert np.abs(l_gpu - f["lhat"]).max() <= 2e-3 * np.sqrt((f["lhat"] ** 2).mean()), "student logits"
    assert abs(s[0] - loss) <= 1e-3 * abs(loss), (s[0], loss)
    # the CE kernel on its own logits (fp64 recomputation of R34 from the GPU's fp32 values)
    t32 = (tl.cpu() + b.cpu()).double().numpy()
    l32 = (sl.cpu() + b.cpu()).double().numpy()
    p = O.softmax(t32)
    ce = float(np.sum(np.log(np.exp(l32 - l32.max(1, keepdims=True)).sum(1)) + l32.max(1) - (p * l32).sum(1)))
    assert abs(s[0] - ce) <= 1e-4 * abs(ce), (s[0], ce)
    # fidelity counts: same decision precision on both sides (fp32 logits + fp32 bias)
    hits = O.fidelity_counts((sl.cpu() + b.cpu()).numpy(), (tl.cpu() + b.cpu()).numpy(), sh.k)
    assert tuple(int(v) for v in s[1:]) == hits, (s[1:], hits)
    G1, G2 = g1.double().cpu().numpy(), g2.double().cpu().numpy()
    e1, e2 = _rel(G1, o1), _rel(G2, o2)
    m1 = float(np.abs(G1 - o1).max() / np.sqrt((o1 ** 2).mean()))
    m2 = float(np.abs(G2 - o2).max() / np.sqrt((o2 ** 2).mean()))
    print(name, "loss", s[0], loss, "grad rel err", e1, e2, "max elem err / RMS", m1, m2, "hits", hits, "N", N)
    assert m1 <= 2e-2 and m2 <= 2e-2, (m1, m2)
    rt.close()


def test_distill_apply_update_and_bf16_copy():
    sh, T = CASES["mid-ragged"]
    rt, x, xn, W, b, w1, w2 = _setup(sh, 1)
    m = torch.randn(sh.E, sh.h, device="cuda")
    g = torch.randn(sh.E, sh.h, device="cuda")
    w = torch.empty(sh.E, sh.h, dtype=torch.bfloat16, device="cuda")
    m0 = m.clone()
    rt.distill_apply(m, g, w, -0.37)
    torch.cuda.synchronize()
    ref = m0.double() - 0.37 * g.double()
    assert torch.allclose(m.double(), ref, rtol=1e-6, atol=1e-7)
    assert torch.equal(w, m.to(torch.bfloat16))             # torch's RNE bf16 rounding of the master
    rt.close()


def test_distill_fixed_point_no_drift_zero_residual():
    """x' = x and Ŵ² = 0: student ≡ teacher bit-for-bit (same GEMM, zero extra K), so
    q − p = 0 exactly, every gradient is exactly 0 and the fidelity is (1, 1, 1)."""
    sh, T = CASES["mid-ragged"]
    rt, x, xn, W, b, w1, w2 = _setup(sh, 2, zero_w2=True, same_x=True)
    N = sh.G * T
    g1 = torch.full((sh.h, sh.H), 7.0, device="cuda")
    g2 = torch.full((sh.E, sh.h), 7.0, device="cuda")
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    rt.distill_grad(x, xn, W, b, w1, w2, g1, g2, stats)
    torch.cuda.synchronize()
    assert torch.count_nonzero(g1) == 0 and torch.count_nonzero(g2) == 0
    s = stats.cpu().tolist()
    assert s[1:] == [N * sh.k, N * ((sh.k + 1) // 2), N * sh.k]
    rt.close()


def test_distill_descent_tracks_oracle():
    """Full-batch descent on one batch: the GPU loss trajectory follows the oracle's fp64
    descent (R36) within 1% and decreases monotonically."""
    from paper_2602_00509_b200.distill import PredictorDistiller
    sh, T = CASES["mid-ragged"]
    rt, x, xn, W, b, w1, w2 = _setup(sh, 3, zero_w2=True)
    N = sh.G * T
    d = PredictorDistiller(rt, w1, w2)
    X, XN, Wn, bn = _np(x).reshape(N, sh.H), _np(xn).reshape(N, sh.H), _np(W), _np(b)
    m1, m2 = _np(w1), np.zeros((sh.E, sh.h))
    lr = 2.0
    prev = None
    for it in range(15):
        met = d.step(x, xn, W, b, lr=lr)
        loss, o1, o2, _ = O.distill_grads(X, XN, Wn, bn, O.round_bf16(m1), O.round_bf16(m2))
        assert abs(met["loss"] - loss / N) <= 1e-2 * loss / N, (it, met["loss"], loss / N)
        if prev is not None:
            assert met["loss"] < prev
        prev = met["loss"]
        m1, _ = O.distill_apply(m1, o1, lr, N)
        m2, _ = O.distill_apply(m2, o2, lr, N)
    rt.close()

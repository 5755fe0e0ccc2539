"""Integer planner cost constants from measured B200 peaks (reading R11).

α = F̄/F_peak per routed pair (Eq. 2, F̄ = 6HF), β = 2·2H/BW_net per remote pair (Eq. 4-5
with λ = 1 and dispatch + combine), n_sat = F_peak/BW_HBM (η_g knee: below it a GEMM is
weight-bandwidth bound), BW_net = 770 GB/s measured B200 peer copy (B200_PROFILING.md).
"""
from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BW_NET = 770e9


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def cost_model(H: int, F: int, pk=None):
    """→ (alpha_ps, beta_ps, n_sat, bw_bytes_per_us)."""
    pk = pk or peaks()[0]
    fpeak = pk["bf16_tflops_sustained"] * 1e12
    alpha_ps = int(round(6.0 * H * F / fpeak * 1e12))
    beta_ps = int(round(2 * 2 * H / BW_NET * 1e12))
    n_sat = int(round(fpeak / (pk["hbm_gbs"] * 1e9)))
    return alpha_ps, beta_ps, n_sat, int(BW_NET / 1e6)


def window_ns(H: int, F: int, T: int, k: int, pk=None, E: int = 0, G: int = 0) -> int:
    """Hiding window (R26): modeled expert-GEMM time of a balanced rank, in ns.

    With E and G given, the model is the planner's own cost (R11) of the balanced rank:
    α·Σ_e c(m_e) over its E/G experts, m = T·k·G/E rows each, c(m) = max(m, n_sat) — so a
    decode-sized GEMM (m < n_sat, weight-bandwidth bound) gets its weight-streaming time,
    not its FLOP time (C2: 123 µs instead of 37 µs).  Without them: FLOP time T·k·6HF/F_peak."""
    pk = pk or peaks()[0]
    pairs = T * k
    if E and G:
        _, _, n_sat, _ = cost_model(H, F, pk)
        pairs = (E // G) * max(T * k * G / E, n_sat)
    return int(6.0 * H * F * pairs / (pk["bf16_tflops_sustained"] * 1e12) * 1e9)

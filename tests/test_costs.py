"""Host-side planner cost constants (DESIGN R11) and the hiding-window model (R26)."""
import pytest

from paper_2602_00509_b200.costs import cost_model, window_ns

PK = {"hbm_gbs": 6553.0, "bf16_tflops": 1675.8, "bf16_tflops_sustained": 1393.9}


def test_cost_constants_follow_r11():
    a, b, n, bw = cost_model(2048, 768, PK)
    assert a == round(6 * 2048 * 768 / 1393.9e12 * 1e12)          # α: 6HF FLOP per pair at F_peak, in ps
    assert b == round(2 * 2 * 2048 / 770e9 * 1e12)                # β: 2·2H bytes per remote pair at BW_net
    assert n == round(1393.9e12 / 6553e9)                          # n_sat: F_peak / BW_HBM (η_g knee)
    assert bw == 770_000                                            # bytes per µs


def test_window_prefill_is_flop_time():
    # C1: 4096 rows per local expert ≫ n_sat, so the saturating model equals the FLOP time
    flop = window_ns(2048, 768, 8192, 8, PK)
    assert window_ns(2048, 768, 8192, 8, PK, E=128, G=8) == flop
    assert flop == int(6 * 2048 * 768 * 8192 * 8 / 1393.9e12 * 1e9)


def test_window_decode_is_weight_streaming_time():
    # C2: 64 rows per local expert < n_sat: each of the 16 local experts costs n_sat rows,
    # i.e. its weights' HBM time (𝒲 = 6HF bytes in bf16, / BW_HBM), not its FLOP time
    H = F = 2880
    _, _, n_sat, _ = cost_model(H, F, PK)
    w = window_ns(H, F, 256, 4, PK, E=128, G=8)
    assert w == int(6 * H * F * 16 * n_sat / 1393.9e12 * 1e9)
    assert w > 3 * window_ns(H, F, 256, 4, PK)
    weights_hbm_ns = 16 * 6 * H * F / 6553e9 * 1e9                  # 16 experts' bf16 weights at BW_HBM
    assert w == pytest.approx(weights_hbm_ns, rel=0.01)
    # cap (Eq. 6 with R15): one 49.8 MB replica fits the window at 770 GB/s, two do not
    cap = w * 770_000 // (6 * H * F * 1000)
    assert cap == 1


def test_bench_placement_policies():
    """bench.py's host-side policies: the dedup wire when ranks span processes (NVLink), and the
    fused gate + predictor stage 1 when one process hosts several ranks (HBM-bound dispatch);
    shapes the fused path does not support (E % 32, k > 8) keep the aux-stream predictor."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import probe_inputs as pi
    a = bench.parse_args([])
    assert a.wire == "auto" and a.gate_fuse == "auto"
    assert not bench._wire_dedup(a, 1) and bench._wire_dedup(a, 8)
    assert bench._gate_fuse(a, 8, pi.C1) and bench._gate_fuse(a, 4, pi.C3)
    assert not bench._gate_fuse(a, 1, pi.C1)                       # one rank per GPU: paper's placement
    assert not bench._gate_fuse(a, 2, pi.C0)                       # E = 8: not a multiple of 32
    assert not bench._gate_fuse(a, 8, pi.C1.with_(k=9))            # top-k above the fused select's 8
    assert bench._gate_fuse(bench.parse_args(["--gate-fuse", "1"]), 1, pi.C1)
    assert not bench._gate_fuse(bench.parse_args(["--gate-fuse", "0"]), 8, pi.C1)
    with pytest.raises(SystemExit):
        bench.parse_args(["--warmup", "2"])                        # W >= 3 (timing rules)

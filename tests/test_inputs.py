"""Generator contract: exact bf16, determinism, skew calibration."""
import numpy as np
import torch

import probe_inputs as pi
from oracle import imbalance_ratio


def test_hadamard_orthogonal():
    h = pi.hadamard_rows(64, np.arange(64)).astype(np.int64)
    assert np.array_equal(h @ h.T, 64 * np.eye(64, dtype=np.int64))


def test_x_exact_and_deterministic():
    shape = pi.C0.with_(H=320)       # H > n_h: exercises the noise tail
    a = pi.layer_inputs(shape, step=5, layer=2)
    b = pi.layer_inputs(shape, step=5, layer=2)
    assert torch.equal(a.x.view(torch.int16), b.x.view(torch.int16))
    # every value in [:n_h] is an integer multiple of 1/n_h, |v| ≤ 256/n_h
    v = a.x[..., :shape.n_h].float() * shape.n_h
    assert torch.equal(v, v.round()) and v.abs().max() <= 256
    c = pi.layer_inputs(shape, step=6, layer=2)
    assert not torch.equal(a.x, c.x)                  # hotspots migrate step to step


def test_static_ir_calibration_c1_shape():
    # SURVEY §8(d) calibration: C1 G=8 s=1.0 static-EP IR mean ≈ 1.7 (band 1.43–2.6)
    shape = pi.C1.with_(T=2048)
    irs = []
    for step in range(3):
        loads = np.zeros(shape.G)
        for r in range(shape.G):
            S = pi.draw_routing(shape, step, 0, r, 1.0)
            loads += np.bincount(S.reshape(-1) // (shape.E // shape.G), minlength=shape.G)
        irs.append(imbalance_ratio(loads))
    assert 1.2 < np.mean(irs) < 2.6

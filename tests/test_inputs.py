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


def test_natural_generator_logits_exact_with_ties():
    """Natural generator: logits x·Wᵀ + b exact in fp32 in any summation order
    (fp32 torch matmul == fp64), negative and dense, with exact ties from duplicated router rows."""
    import numpy as np
    import torch
    import probe_inputs as pi
    sh = pi.C0.with_(name="nat", E=64, k=8, H=2048, F=64, T=256, G=1)
    W, b = pi.natural_router(sh, 0, 0, 1.2)
    x = pi.natural_layer_inputs(sh, 0, 0).x[0]
    l64 = pi.bf16_to_numpy_f64(x) @ pi.bf16_to_numpy_f64(W).T + b.double().numpy()[None, :]
    l32 = (x.float() @ W.float().T + b[None, :]).double().numpy()
    l32r = (x.float().flip(1) @ W.float().flip(1).T + b[None, :]).double().numpy()   # another order
    assert np.array_equal(l64, l32) and np.array_equal(l64, l32r)
    assert (l64 < 0).mean() > 0.3
    srt = np.sort(l64, axis=1)[:, ::-1]
    assert (srt[:, 0] == srt[:, 1]).any() or (l64[:, :, None] == l64[:, None, :]).sum() > l64.size

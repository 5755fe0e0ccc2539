"""GPU: CUDA-Graph capture of one full dual-track layer step ("maintaining CUDA
Graph capture compatibility"): forward(L) on the capture stream, predict/plan(L+1) on the
aux stream, split-phase prefetch(L+1) on the prefetch stream, joined back by the
prefetch WAIT.  Replays must reproduce eager execution bit-for-bit (every kernel is
deterministic; the GEMM tile scheduler is dynamic but each tile's arithmetic is fixed)."""
import pytest
import torch

import probe_inputs as pi

pytestmark = pytest.mark.gpu


def _setup(sh):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    cfg = ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=sh.F, T=sh.T, h=sh.h, alpha_ps=1, beta_ps=0)
    rt = ProbeRuntime(cfg)
    dev = "cuda"
    L = [pi.layer_inputs(sh, 0, i, 1.5, device=dev, wrap=4) for i in range(3)]
    W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
    ex = [pi.expert_weights(sh, p, device=dev) for p in (0, 1)]
    res = [pi.predictor_residual(sh, p, device=dev) for p in (0, 1)]
    win = torch.full((sh.G,), 10 ** 9, dtype=torch.int64, device=dev)
    return rt, L, W, ex, res, win


def _step(rt, L, W, ex, res, win, layer, out, stream):
    p, q = layer % 2, (layer + 1) % 2
    rt.forward(layer, L[layer].x, W[p], None, ex[p][0], ex[p][1], out, use_plan=layer > 0, stream=stream)
    rt.predict(layer + 1, L[layer].x, W[q], None, res[q][0], res[q][1])
    rt.plan(layer + 1, win)
    rt.prefetch(layer + 1, ex[q][0], ex[q][1], phase=0)
    rt.prefetch(layer + 1, phase=1, stream=stream)      # join the prefetch stream back


def test_graph_capture_replay_matches_eager():
    sh = pi.C0.with_(name="graph", E=32, k=4, H=256, F=256, T=96, G=4)
    s = torch.cuda.Stream()
    # eager reference
    rt, L, W, ex, res, win = _setup(sh)
    out_e = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    with torch.cuda.stream(s):
        _step(rt, L, W, ex, res, win, 0, out_e, s)
        _step(rt, L, W, ex, res, win, 1, out_e, s)
    torch.cuda.synchronize()
    ref = out_e.clone()
    rt.close()
    # captured: layer 0 eager (warm-up, plans layer 1), layer 1 captured and replayed
    rt, L, W, ex, res, win = _setup(sh)
    out_g = torch.empty(sh.G, sh.T, sh.H, device="cuda")
    with torch.cuda.stream(s):
        _step(rt, L, W, ex, res, win, 0, out_g, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _step(rt, L, W, ex, res, win, 1, out_g, s)
    for _ in range(3):
        out_g.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_g, ref)
    rt.check()
    rt.close()

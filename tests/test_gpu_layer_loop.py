"""NEXT-2 ("Mandating CUDA Graph Compatibility"): the whole multi-layer
loop — a DP-attention window before every MoE layer, the main track, the aux track
(predict / plan of L+1) and the split-phase prefetch — captured as ONE CUDA graph and replayed,
with EVERY layer of every replay checked against the fp64 oracle: routing ids bit-exact, gate
weights 1e-6, layer outputs within 2e-2·RMS.  Layer L+1 runs on the plan made from the
prediction computed during layer L, exactly as in serving.

The attention stand-in (QKV / O projections + causal GQA SDPA, torch library kernels, not part
of the PROBE path) provides the window the split-phase part 2 hides behind; its output is not
fed to the MoE, whose inputs are the designed routing inputs (exact, comparable routing).
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import probe_inputs as pi
from layer_harness import LazyExperts, f64

pytestmark = pytest.mark.gpu

POOL = 4


@pytest.mark.parametrize("dedup,fused", [(False, False), (True, False), (False, True)])
def test_graph_layer_loop_every_layer_matches_oracle(dedup, fused):
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    sh = pi.C0.with_(name="loop", E=32, k=4, H=256, F=256, T=128, G=4)
    G, E, k, H, T = sh.G, sh.E, sh.k, sh.H, sh.T
    cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=sh.F, T=T, h=sh.h, alpha_ps=1, beta_ps=0, dedup_wire=dedup,
                      predispatch=dedup, fuse_gate_predictor=fused)
    rt = ProbeRuntime(cfg)
    dev = "cuda"
    pool = [pi.layer_inputs(sh, 0, i, 1.3, device=dev, wrap=POOL) for i in range(POOL)]
    W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
    ex = [pi.expert_weights(sh, p, device=dev) for p in (0, 1)]
    res = [pi.predictor_residual(sh, p, device=dev) for p in (0, 1)]
    win = torch.full((G,), 10 ** 9, dtype=torch.int64, device=dev)
    outs = [torch.empty(G, T, H, device=dev) for _ in range(POOL)]
    ids = [torch.empty(G, T, k, dtype=torch.int32, device=dev) for _ in range(POOL)]
    gws = [torch.empty(G, T, k, dtype=torch.float32, device=dev) for _ in range(POOL)]
    nq, nkv, hd = 4, 2, 64
    g = torch.Generator(device="cpu").manual_seed(3)
    wq = (torch.randn(nq * hd, H, generator=g) / H ** 0.5).to(torch.bfloat16).to(dev)
    wkv = (torch.randn(2 * nkv * hd, H, generator=g) / H ** 0.5).to(torch.bfloat16).to(dev)
    wo = (torch.randn(H, nq * hd, generator=g) / (nq * hd) ** 0.5).to(torch.bfloat16).to(dev)
    attn_sink = torch.empty(G * T, H, dtype=torch.bfloat16, device=dev)
    s = torch.cuda.Stream()

    def attention(x):
        x2 = x.reshape(-1, H)
        q = (x2 @ wq.T).view(G, T, nq, hd).transpose(1, 2)
        kv = (x2 @ wkv.T).view(G, T, 2, nkv, hd)
        kk, vv = kv[:, :, 0].transpose(1, 2), kv[:, :, 1].transpose(1, 2)
        o = F.scaled_dot_product_attention(q, kk, vv, is_causal=True, enable_gqa=True)
        torch.matmul(o.transpose(1, 2).reshape(-1, nq * hd), wo.T, out=attn_sink)

    def loop(L0):
        for L in range(L0, L0 + POOL):
            i, p, q = L % POOL, L % 2, (L + 1) % 2
            attention(pool[i].x)
            if fused:        # layer L's gate GEMM also computes stage 1 of layer L+1's predictor
                rt.predict_prepare(L + 1, W[q], res[q][0])
            rt.forward(L, pool[i].x, W[p], None, ex[p][0], ex[p][1], outs[i], use_plan=L > 0, topk_ids=ids[i],
                       topk_w=gws[i], stream=s)
            rt.predict(L + 1, pool[i].x, W[q], None, res[q][0], res[q][1])
            rt.plan(L + 1, win)
            rt.prefetch(L + 1, ex[q][0], ex[q][1], phase=0)
        rt.prefetch(L0 + POOL, phase=1, stream=s)          # join the aux / prefetch streams

    # oracle for the captured layers 4..7 (same inputs as 0..3; layer L uses the plan predicted in L-1)
    W64 = [f64(w) for w in W]
    r64 = [(f64(a), f64(b)) for a, b in res]
    pcfg = O.PlannerConfig(G=G, E=E, replica_budget=3, kmax=16, alpha_ps=1, beta_ps=0, n_sat=0,
                           bw_bytes_per_us=770_000, expert_bytes=3 * H * sh.F * 2)
    refs = {}
    for L in range(POOL, 2 * POOL):
        xs = [f64(pool[L % POOL].x[r]) for r in range(G)]
        xp = [f64(pool[(L - 1) % POOL].x[r]) for r in range(G)]
        nhat = np.stack([O.predict_counts(xp[r], W64[L % 2], None, *r64[L % 2], k)[0] for r in range(G)])
        plan = O.plan_greedy(nhat, [10 ** 9] * G, pcfg)
        refs[L % POOL] = O.layer_reference(xs, W64[L % 2], None, k, plan, G, E, LazyExperts(ex[L % 2][0]),
                                           LazyExperts(ex[L % 2][1]))

    def check(tag):
        torch.cuda.synchronize()
        for i in range(POOL):
            ref = refs[i]
            got_ids = ids[i].cpu().numpy()
            rms = np.sqrt(np.mean(np.concatenate([o.reshape(-1) for o in ref["out"]]) ** 2))
            for r in range(G):
                assert np.array_equal(got_ids[r], ref["ids"][r]), f"{tag}: ids layer {i} rank {r}"
                assert np.abs(gws[i][r].cpu().numpy() - ref["g"][r]).max() < 1e-6, f"{tag}: gate weights {i}"
                err = np.abs(outs[i][r].cpu().numpy() - ref["out"][r]).max()
                assert err <= 2e-2 * rms, f"{tag}: output layer {i} rank {r}: {err} > 2e-2 * {rms}"

    with torch.cuda.stream(s):
        loop(0)                                              # eager warm-up: layer 0 static, plans 1..4
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        loop(POOL)                                           # layers 4..7 (+ plan / prefetch of 8 ≡ 4)
    for rep in range(3):
        for o in outs:
            o.zero_()
        for t in ids:
            t.fill_(-1)
        graph.replay()
        check(f"replay {rep}")
    rt.check()
    if dedup:
        assert rt.flags()[5] > 0                             # pre-dispatch hits inside the graph
    rt.close()

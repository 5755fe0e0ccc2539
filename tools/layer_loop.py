"""Whole-layer loop with a DP-attention window, captured as one CUDA graph (
P:229-232 CUDA-Graph compatibility, "the remaining transfers are hidden behind the
attention computation of the next layer").

Each layer = attention stand-in (QKV / output projections + causal GQA SDPA on the rank's own
tokens, Qwen3-30B-A3B-shaped: 32 query heads, 4 KV heads, head dim 128; library kernels, not
part of the PROBE path) followed by the PROBE MoE layer (forward(L) on the main stream,
predict/plan(L+1) on the aux stream, split-phase prefetch(L+1) on the prefetch stream).  The
attention output is discarded: the MoE inputs are the designed routing inputs, so the timing
is of the real kernels while routing stays exact.

Reports per-layer ms for: attention alone, MoE alone, the loop eagerly, the loop as one CUDA
graph (PROBE and static EP), and the exposed prefetch wait from the library's phase profile.

  python tools/layer_loop.py --layers 8 --reps 5
"""
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import probe_inputs as pi  # noqa: E402
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime  # noqa: E402
from paper_2602_00509_b200._lib import PHASES  # noqa: E402
from paper_2602_00509_b200.costs import cost_model, window_ns  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seq", type=int, default=2048, help="attention sequence length (T per rank = batch · seq)")
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--gate-fuse", type=int, default=1, help="fused gate + predictor stage 1 (bench.py's 1-GPU default)")
    a = ap.parse_args()
    sh = pi.C1
    dev = torch.device("cuda", 0)
    G, T, H, F_, E = sh.G, sh.T, sh.H, sh.F, sh.E
    al, be, ns, bw = cost_model(H, F_)
    rt = ProbeRuntime(ProbeConfig(G=G, E=E, k=sh.k, H=H, F=F_, T=T, h=sh.h, alpha_ps=al, beta_ps=be, n_sat=ns,
                                  bw_bytes_per_us=bw, capacity_factor=4.0,
                                  fuse_gate_predictor=bool(a.gate_fuse)), dev)
    POOL = 4
    pool = [pi.layer_inputs(sh, 0, i, a.zipf, device=dev, wrap=POOL) for i in range(POOL)]
    W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
    ex = [pi.expert_weights(sh, p, device=dev) for p in (0, 1)]
    res = [pi.predictor_residual(sh, p, device=dev) for p in (0, 1)]
    win = torch.full((G,), window_ns(H, F_, T, sh.k, E=sh.E, G=G), dtype=torch.int64, device=dev)
    out = torch.empty(G, T, H, device=dev)
    # attention stand-in weights (Qwen3-30B-A3B attention shapes)
    nq, nkv, hd = 32, 4, 128
    g = torch.Generator(device="cpu").manual_seed(7)
    wq = (torch.randn(nq * hd, H, generator=g) / H ** 0.5).to(torch.bfloat16).to(dev)
    wk = (torch.randn(nkv * hd, H, generator=g) / H ** 0.5).to(torch.bfloat16).to(dev)
    wv = (torch.randn(nkv * hd, H, generator=g) / H ** 0.5).to(torch.bfloat16).to(dev)
    wo = (torch.randn(H, nq * hd, generator=g) / (nq * hd) ** 0.5).to(torch.bfloat16).to(dev)
    attn_out = torch.empty(G * T, H, dtype=torch.bfloat16, device=dev)
    B = G * T // a.seq

    def attention(x):
        x2 = x.reshape(-1, H)
        q = (x2 @ wq.T).view(B, a.seq, nq, hd).transpose(1, 2)
        k = (x2 @ wk.T).view(B, a.seq, nkv, hd).transpose(1, 2)
        v = (x2 @ wv.T).view(B, a.seq, nkv, hd).transpose(1, 2)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        torch.matmul(o.transpose(1, 2).reshape(-1, nq * hd), wo.T, out=attn_out)

    main_s = torch.cuda.Stream(dev)

    def layer(L, use_plan=True, attn=True, moe=True):
        li = pool[L % POOL]
        p, q = L % 2, (L + 1) % 2
        if attn:
            attention(li.x)
        if moe:
            if use_plan and a.gate_fuse:
                rt.predict_prepare(L + 1, W[q], res[q][0])
            rt.forward(L, li.x, W[p], None, ex[p][0], ex[p][1], out, use_plan=use_plan and L > 0, stream=main_s)
            if use_plan:
                rt.predict(L + 1, li.x, W[q], None, res[q][0], res[q][1])
                rt.plan(L + 1, win)
                rt.prefetch(L + 1, ex[q][0], ex[q][1], phase=0)

    def loop(L0, n, **kw):
        for i in range(n):
            layer(L0 + i, **kw)
        if kw.get("use_plan", True) and kw.get("moe", True):
            rt.prefetch(L0 + n, phase=1, stream=main_s)      # join the prefetch stream (graph-safe end)

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(main_s)
        for _ in range(reps):
            fn()
        e1.record(main_s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    n = a.layers
    assert n % 4 == 0, "layers per loop must be a multiple of the input-pool period (4) for graph replays"
    res_out = {"config": {"shape": "C1", "G": G, "T": T, "layers_per_loop": n, "gate_fused_predictor": bool(a.gate_fuse),
                          "attention": f"{B}x{a.seq} tokens, "
                          f"{nq} q heads / {nkv} kv heads / hd {hd}, causal SDPA + projections (torch library)"}}
    state = {"L": 0}

    def next_loop(**kw):
        L0 = state["L"]
        loop(L0, n, **kw)
        state["L"] = L0 + n

    with torch.cuda.stream(main_s):
        next_loop()                                          # warm-up (layer 0 static, plans from layer 1)
        torch.cuda.synchronize()
        res_out["attention_only_ms"] = timed(lambda: loop(0, n, moe=False), a.reps) / n
        res_out["moe_only_ms"] = timed(lambda: next_loop(attn=False), a.reps) / n
        res_out["loop_eager_ms"] = timed(next_loop, a.reps) / n
        # exposed prefetch wait inside the loop (library phase profile, eager)
        rt.profile(n)
        next_loop()
        torch.cuda.synchronize()
        ph = rt.profile_read()
        rt.profile(0)
        res_out["phases_ms_in_loop"] = {nm: float(ph[:, i].mean()) for i, nm in enumerate(PHASES)}
        # the whole loop (attention + MoE + aux + prefetch streams) as one CUDA graph; replays
        # re-run the same layer numbers, whose plans / slot banks repeat with period n
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=main_s):
            loop(state["L"], n)
        res_out["loop_graph_ms"] = timed(graph.replay, a.reps) / n
        state["L"] += n
        # static EP with the same attention window, eager and as a graph
        res_out["static_loop_eager_ms"] = timed(lambda: next_loop(use_plan=False), a.reps) / n
        sgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(sgraph, stream=main_s):
            loop(state["L"], n, use_plan=False)
        res_out["static_loop_graph_ms"] = timed(sgraph.replay, a.reps) / n
    rt.check()
    print(json.dumps(res_out))
    rt.close()


if __name__ == "__main__":
    main()

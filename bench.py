#!/usr/bin/env python
"""bench.py — PROBE expert-parallel MoE layer (dynamic replication) on B200.

One step = one pass of the whole hot path over one batch: the main
track of layer L (gate → count all-gather → materialize plan(L) → dispatch →
grouped SwiGLU GEMMs → combine) with the auxiliary track for L+1 (lookahead
predictor → balance planner → split-phase replica prefetch) running beside it.
Layers alternate parity; inputs cycle through a pool of Hadamard-encoded
Zipf-skewed layers whose hotspots migrate layer to layer.

Default workload: BASELINE.json configs[1] (Qwen3-30B-A3B-shaped: E=128, k=8,
H=2048, F=768, 8192 tokens per rank, EP=8).  With --gpus N the G=8 logical EP
ranks are spread over N GPUs (G/N per process); at N=1 all eight ranks run on
one B200 (single-GPU EP emulation: every peer pointer is local HBM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl probe|reference]
                    [--config C1|C2|C3] [--zipf S]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import probe_inputs as pi  # noqa: E402

METRIC_PREFILL = "MoE-layer prefill latency (ms)"
METRIC_DECODE = "MoE-layer decode throughput (tokens/s)"
POOL = 4            # distinct layer inputs cycled (each > L2: 268 MB of x at C1)


from paper_2602_00509_b200.costs import cost_model as _cost_model, peaks, window_ns  # noqa: E402


def cost_model(shape, pk):
    return _cost_model(shape.H, shape.F, pk)


class ClockSampler:
    """SM clock / clock-event-reason sampling DURING the timed region (B200_PROFILING.md).

    NVML from a background thread every 2 ms (the timed region of a C1 run is ~0.1 s, too
    short for `nvidia-smi -lms`, whose first sample arrives after process start-up); falls
    back to nvidia-smi when NVML is unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index=0, period_s=0.002):
        self.gpu, self.period = gpu_index, period_s
        self.sm, self.mask, self.max_sm = [], 0, None
        self.h = None
        self.smi = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            idx = torch.cuda._get_nvml_device_index(self.gpu)
        except Exception:
            idx = self.gpu
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def __enter__(self):
        import threading
        try:
            nv, h = self._nvml_handle()
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.stop = threading.Event()

            def loop():
                while not self.stop.is_set():
                    try:
                        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        self.mask |= int(reasons(h))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
            self.h = h
        except Exception:
            self.h = None
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.smi = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm",
                     "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:
                self.smi = None
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.th.join(timeout=2)
        if self.smi is not None:
            self.smi.terminate()
            try:
                self.smi.wait(timeout=5)
            except Exception:
                self.smi.kill()
            try:
                for r in open(self.f.name).read().split("\n"):
                    c = r.split(",")
                    if len(c) >= 2 and c[0].strip().replace(".", "").isdigit():
                        self.sm.append(float(c[0]))
                        self.max_sm = float(c[1])
            except Exception:
                pass

    def summary(self):
        reasons = sorted(n for bit, n in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(self.sm), "source": "nvml" if self.h is not None else "nvidia-smi"}


# =============================================================================
# PROBE arm
# =============================================================================

def run_probe(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (launch N>1 with torchrun)")
    # PROBE_BENCH_SHARED_GPU=1: functional check of the N>1 path on a one-GPU box — every rank
    # on cuda:0 over gloo (NCCL refuses two ranks on one device); never a performance number
    shared = os.environ.get("PROBE_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    env = dict(world=world, rank=rank, local=local, shared=shared, dev=dev, pg=pg)
    shape = pi.SHAPES[args.config]
    if args.ep:
        shape = shape.with_(G=args.ep)
    result = measure(shape, args, env, light=False)
    if world == 1 and not args.no_dedup_sub and result is not None and args.wire != "dedup":
        # the dedup wire format (one row per unique (token, dest), R25 partial combine) on the same
        # inputs: the NVLink-product format, measured here with every "remote" row in local HBM
        result["dedup_wire"] = measure(shape, args, env, light=True, dedup=True)
        # NEXT-4 predictive pre-dispatch on top of the dedup wire (overlaps the wire with the gate)
        result["predispatch"] = measure(shape, args, env, light=True, dedup=True, predispatch=True)
    if args.config == "C1" and not args.no_decode:
        # BASELINE.json's metric has two halves: prefill latency (C1, this line's value) and
        # decode tokens/s (C2, GPT-OSS-120B-shaped, batch 256 per rank) — measured in the same run
        dec = measure(pi.C2.with_(G=shape.G), args, env, light=True)
        if result is not None:
            result["decode"] = dec
    if result is not None:
        print(json.dumps(result), flush=True)
    if pg is not None:
        torch.distributed.destroy_process_group()
    return result


def _wire_dedup(args, world):
    """Wire format of the headline measurement: `--wire auto` uses the dedup format (one row per
    unique (token, destination), D6) when the ranks span processes — i.e. GPUs joined by NVLink —
    and the per-slot rows (D1) when one process hosts every rank (all "remote" rows are local HBM)."""
    return args.wire == "dedup" or (args.wire == "auto" and world > 1)


def _gate_fuse(args, GL, shape):
    """`--gate-fuse auto`: the gate GEMM of layer L also computes layer L+1's prior logits and
    predictor activation (x read once, probe_config.fuse_gate_predictor) when several logical ranks
    share this GPU — their dispatch is HBM-bound and an aux-stream predictor re-reading x slows it.
    With one rank per GPU the NVLink dispatch leaves the SMs idle and hides the aux-stream predictor
    (P:467), so the paper's placement stays."""
    ok = shape.E % 32 == 0 and shape.k <= 8
    if args.gate_fuse == "auto":
        return ok and GL > 1
    return ok and args.gate_fuse == "1"


def measure(shape, args, env, light=False, dedup=None, predispatch=False):
    """Bench one configuration: PROBE (timed, profiled), static EP, and unless `light` the
    EP emulation, e2e, roofline and CPU baseline.  Rank 0 returns the JSON dict (else None)."""
    from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime
    from paper_2602_00509_b200._lib import PHASES
    world, rank, local, shared, dev, pg = (env[k] for k in ("world", "rank", "local", "shared", "dev", "pg"))
    G = shape.G
    if G % world:
        raise SystemExit(f"EP={G} ranks cannot be spread over {world} GPUs")
    GL = G // world
    R0 = rank * GL
    pk, pk_kind = peaks()
    alpha_ps, beta_ps, n_sat, bw_Bpus = cost_model(shape, pk)
    cfg = ProbeConfig(G=G, E=shape.E, k=shape.k, H=shape.H, F=shape.F, T=shape.T, h=shape.h, rank_begin=R0,
                      local_ranks=GL, replica_budget=3, kmax=16, n_sat=n_sat, alpha_ps=alpha_ps, beta_ps=beta_ps,
                      bw_bytes_per_us=bw_Bpus, capacity_factor=args.cap if G > 1 else 1.0,
                      dedup_wire=(_wire_dedup(args, world) if dedup is None else dedup) or predispatch,
                      predispatch=predispatch, fuse_gate_predictor=_gate_fuse(args, GL, shape))
    if world > 1:
        from paper_2602_00509_b200.dist import make_runtime_distributed
        rt = make_runtime_distributed(cfg, dev, pg)
    else:
        rt = ProbeRuntime(cfg, dev)
    if args.aux_sms:
        from paper_2602_00509_b200._lib import OPT_AUX_SMS
        rt.set_option(OPT_AUX_SMS, args.aux_sms)
    if args.aux_start:
        from paper_2602_00509_b200._lib import OPT_AUX_START
        rt.set_option(OPT_AUX_START, args.aux_start)
    if args.pred_pair is not None:
        from paper_2602_00509_b200._lib import OPT_PRED_PAIR
        rt.set_option(OPT_PRED_PAIR, args.pred_pair)
    if args.l2hint:
        from paper_2602_00509_b200._lib import OPT_L2_HINTS
        rt.set_option(OPT_L2_HINTS, args.l2hint)
    if args.epi_topk:
        from paper_2602_00509_b200._lib import OPT_FUSED_EPILOGUE_TOPK
        rt.set_option(OPT_FUSED_EPILOGUE_TOPK, 1)
    if args.pred_maxreg:
        from paper_2602_00509_b200._lib import OPT_PRED_MAXREG
        rt.set_option(OPT_PRED_MAXREG, args.pred_maxreg)
    ranks = list(range(R0, R0 + GL))
    t0 = time.time()
    key = (shape, args.zipf, tuple(ranks))
    if env.get("pool_key") != key:          # generated once per configuration (reused by sub-measurements)
        env["pool"] = None
        env["pool"] = [pi.layer_inputs(shape, 0, i, args.zipf, ranks=ranks, device=dev, wrap=POOL) for i in range(POOL)]
        env["pool_key"] = key
    pool = env["pool"]
    W = [pi.router_weight(shape, p, device=dev) for p in (0, 1)]
    experts = list(range(R0 * shape.E // G, (R0 + GL) * shape.E // G))
    w13, w2 = [], []
    for p in (0, 1):
        a, b = pi.expert_weights(shape, p, experts=experts, device=dev)
        w13.append(a)
        w2.append(b)
    res = [pi.predictor_residual(shape, p, device=dev) for p in (0, 1)]
    gen_s = time.time() - t0
    T, H = shape.T, shape.H
    # layer output fp32 (R25 "output fp32 for parity": the configuration tests/test_gpu_fullsize.py
    # checks at 2e-2·RMS); --out-bf16 writes the model's activation dtype instead (half the combine
    # writes and e2e D2H bytes; its own rounding reaches ≈1.6e-2·RMS at full size)
    out = torch.empty(GL, T, H, dtype=torch.bfloat16 if args.out_bf16 else torch.float32, device=dev)
    # hiding window (R26): modeled per-rank expert-GEMM time at the balanced load
    gemm_ns = window_ns(H, shape.F, T, shape.k, pk, E=shape.E, G=G)
    win = torch.full((G,), gemm_ns, dtype=torch.int64, device=dev)
    main = torch.cuda.current_stream(dev)

    def step(L, use_plan=True, x=None, fwd_plan=None):
        li = pool[L % POOL]
        p = L % 2
        q = (L + 1) % 2
        xx = li.x if x is None else x
        fp = (use_plan and L > 0) if fwd_plan is None else fwd_plan
        if use_plan and cfg.fuse_gate_predictor:
            rt.predict_prepare(L + 1, W[q], res[q][0])
        rt.forward(L, xx, W[p], None, w13[p], w2[p], out, use_plan=fp)
        if use_plan:
            rt.predict(L + 1, xx, W[q], None, res[q][0], res[q][1])
            if not args.modeled_window:     # R26: last measured GEMM window of every rank (+ attention)
                rt.window(win, attention_ns=args.attn_ns, fallback_ns=gemm_ns)
            rt.plan(L + 1, win)
            rt.prefetch(L + 1, w13[q], w2[q], phase=0)

    def barrier():
        if pg is not None:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def timed(nsteps, L0, use_plan=True, x_host=None, out_host=None, x_dev=None):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(main)
        L = L0
        for _ in range(nsteps):
            if x_host is not None:
                x_dev.copy_(x_host[L % POOL], non_blocking=True)
                step(L, use_plan, x=x_dev)
                out_host.copy_(out, non_blocking=True)
            else:
                step(L, use_plan)
            L += 1
        ev1.record(main)
        barrier()
        ms = ev0.elapsed_time(ev1) / nsteps
        if pg is not None:
            t = torch.tensor([ms], device="cpu" if shared else dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, L

    # ---- warm-up (layer 0 is static: nothing predicts it, R29)
    L = 0
    for _ in range(args.warmup):
        step(L)
        L += 1
    torch.cuda.synchronize(dev)
    rt.check()
    # ---- timed region (PROBE)
    launches0 = rt.launches()
    pf0 = rt.prefetch_kib()
    fl0 = rt.flags()
    with ClockSampler(local) as clk:
        ms, L = timed(args.steps, L)
    launches = rt.launches() - launches0
    pf1 = rt.prefetch_kib()
    fl1 = rt.flags()
    pred_disp = None
    if predispatch:
        hits, miss = fl1[5] - fl0[5], fl1[6] - fl0[6]
        pred_disp = {"pairs_predispatched_hit": hits, "pairs_shipped_after_gate": miss,
                     "hit_rate": hits / max(1, hits + miss),
                     "note": "(token, dest) pairs whose x row was pushed to the home rank of a predicted expert "
                             "during the gate (NEXT-4, P:586) vs shipped by the dispatch after the gate"}
    prefetch = {"part1_MB_per_layer": (pf1[0] - pf0[0]) / 1024 / args.steps,
                "part2_MB_per_layer": (pf1[1] - pf0[1]) / 1024 / args.steps,
                "note": "replica weights pushed by this process: part 1 beside the expert GEMMs, part 2 after "
                        "the combine (split phase, P:469)"}
    clocks = clk.summary()
    torch.cuda.synchronize(dev)
    win_used = [int(v) for v in win.cpu()]
    caps = [int(min(3, (w * bw_Bpus) // (cfg.expert_bytes * 1000))) for w in win_used]
    window_rep = {"source": "modeled" if args.modeled_window else "measured (probe_window, R26)",
                  "window_ns": win_used, "caps": caps, "modeled_ns": gemm_ns, "attention_ns": args.attn_ns}
    # ---- per-phase profile (separate pass; CUDA events on the launching stream)
    rt.profile(args.steps)
    ms_prof, L = timed(args.steps, L)
    ph = rt.profile_read()
    phases = {n: float(ph[:, i].mean()) for i, n in enumerate(PHASES)}
    rt.profile(0)
    # ---- diagnostic layer pair (untimed): planner stats, predicted vs actual load, balance
    pc = torch.empty(G, shape.E, dtype=torch.int32, device=dev)
    pst = torch.empty(8, dtype=torch.int64, device=dev)
    li = pool[L % POOL]
    p, q = L % 2, (L + 1) % 2
    if cfg.fuse_gate_predictor:
        rt.predict_prepare(L + 1, W[q], res[q][0])
    rt.forward(L, li.x, W[p], None, w13[p], w2[p], out, use_plan=True)
    rt.predict(L + 1, li.x, W[q], None, res[q][0], res[q][1], pred_counts=pc)
    rt.plan(L + 1, win, stats=pst)
    rt.prefetch(L + 1, w13[q], w2[q], phase=0)
    L += 1
    step(L)
    L += 1
    counts = torch.empty(G, shape.E, dtype=torch.int32, device=dev)
    split = torch.empty(G, shape.E, G, dtype=torch.int32, device=dev)
    reps = torch.empty(G, 3, dtype=torch.int32, device=dev)
    route = torch.empty(GL, T, shape.k, 2, dtype=torch.int32, device=dev)
    rt.debug_layout(counts, split, route, None, reps)
    torch.cuda.synchronize(dev)
    # wire rows of this layer (one GPU: all "remote" rows are local HBM): per routed (token, slot),
    # per unique (token, destination) — §8(d)'s dispatch/combine unit — and the remote ones
    rd = route[..., 0].long().cpu().numpy()
    valid = route[..., 1].cpu().numpy() >= 0
    srt = np.sort(np.where(valid, rd, -1), axis=2)
    uniq = (srt >= 0) & np.concatenate([np.ones(srt.shape[:2] + (1,), bool), srt[..., 1:] != srt[..., :-1]], axis=2)
    src = np.arange(R0, R0 + GL)[:, None, None]
    wire = {"rows_per_slot": int(valid.sum()), "rows_unique_token_dest": int(uniq.sum()),
            "rows_unique_remote": int((uniq & (srt != src)).sum()), "dedup_wire": bool(cfg.dedup_wire)}
    EL = shape.E // G
    n = counts.cpu().numpy().astype(np.int64)
    nh = pc.cpu().numpy().astype(np.int64)
    stats = pst.cpu().numpy().tolist()
    sc = split.cpu().numpy().astype(np.int64)
    sp = np.diff(np.concatenate([np.zeros((G, shape.E, 1), np.int64), sc], axis=2), axis=2)
    pre = n.sum(axis=0).reshape(G, EL).sum(axis=1)
    post = sp.sum(axis=(0, 1))
    ir_pre = float(pre.max() / pre.mean())
    ir_post = float(post.max() / post.mean())
    nrep = int((reps >= 0).sum().item())
    load_fidelity = float(np.minimum(nh, n).sum() / max(1, n.sum()))
    # ---- static-EP baseline (same library, replication disabled, no aux track)
    for _ in range(2):
        step(L, use_plan=False)
        L += 1
    ms_static, L = timed(args.steps, L, use_plan=False)
    rt.profile(args.steps)
    _, L = timed(args.steps, L, use_plan=False)
    phs = rt.profile_read()
    static_phases = {n: float(phs[:, i].mean()) for i, n in enumerate(PHASES)}
    rt.profile(0)
    # ---- single-GPU EP straggler emulation: expert GEMMs partitioned by logical rank
    #      (~#SMs/G SMs per rank ⇒ GEMM time = the straggler's, Eq. 3); static EP vs PROBE
    ep_em = None
    if world == 1 and GL > 1 and not args.no_emulation and not light:
        from paper_2602_00509_b200._lib import OPT_EP_EMULATION
        rt.set_option(OPT_EP_EMULATION, 1)
        for _ in range(2):
            step(L, use_plan=False)
            L += 1
        ms_em_static, L = timed(args.steps, L, use_plan=False)
        step(L, fwd_plan=False)
        L += 1
        step(L)
        L += 1
        ms_em_probe, L = timed(args.steps, L)
        rt.set_option(OPT_EP_EMULATION, 0)
        ep_em = {"static_ep_ms": ms_em_static, "probe_ms": ms_em_probe,
                 "speedup_probe_vs_static": ms_em_static / ms_em_probe,
                 "note": "expert GEMMs split into G CTA sets (one per logical rank, ~148/G SMs each); "
                         "gate/dispatch/combine unpartitioned"}
        step(L, fwd_plan=False)
        L += 1
    # ---- end-to-end through the API with host buffers (pinned), copies inside the timed region.
    #      Every step copies its input x H2D and its output D2H; the copies run on their own
    #      streams (double-buffered device x / out, host out) so step L's D2H and step L+1's
    #      H2D overlap step L+1's compute, as a serving pipeline would.
    e2e = None
    if not args.no_e2e and not light:
        x_host = [pool[i].x.cpu().pin_memory() for i in range(POOL)]
        NB = 2
        x_dev = [torch.empty_like(pool[0].x) for _ in range(NB)]
        o_dev = [torch.empty_like(out) for _ in range(NB)]
        o_host = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(NB)]
        h2d, d2h, auxs = (torch.cuda.Stream(dev) for _ in range(3))
        step(L, fwd_plan=False)           # re-enter the planned pipeline after the static pass
        L += 1
        step(L)
        L += 1

        def timed_e2e(nsteps, L):
            x_free = [[] for _ in range(NB)]
            o_free = [[] for _ in range(NB)]
            barrier()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(main)
            h2d.wait_stream(main)
            last = []
            for _ in range(nsteps):
                bsel = L % NB
                p, q = L % 2, (L + 1) % 2
                for e in x_free[bsel]:
                    h2d.wait_event(e)
                with torch.cuda.stream(h2d):
                    x_dev[bsel].copy_(x_host[L % POOL], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(h2d)
                main.wait_event(ev_in)
                for e in o_free[bsel]:
                    main.wait_event(e)
                if cfg.fuse_gate_predictor:
                    rt.predict_prepare(L + 1, W[q], res[q][0])
                rt.forward(L, x_dev[bsel], W[p], None, w13[p], w2[p], o_dev[bsel], use_plan=True)
                rt.predict(L + 1, x_dev[bsel], W[q], None, res[q][0], res[q][1], stream=auxs)
                if not args.modeled_window:
                    rt.window(win, attention_ns=args.attn_ns, fallback_ns=gemm_ns, stream=auxs)
                rt.plan(L + 1, win, stream=auxs)
                rt.prefetch(L + 1, w13[q], w2[q], phase=0)
                e_main, e_aux = torch.cuda.Event(), torch.cuda.Event()
                e_main.record(main)
                e_aux.record(auxs)
                x_free[bsel] = [e_main, e_aux]
                d2h.wait_event(e_main)
                with torch.cuda.stream(d2h):
                    o_host[bsel].copy_(o_dev[bsel], non_blocking=True)
                e_out = torch.cuda.Event()
                e_out.record(d2h)
                o_free[bsel] = [e_out]
                last = [e_out, e_aux]
                L += 1
            for e in last:
                main.wait_event(e)
            ev1.record(main)
            barrier()
            ms = ev0.elapsed_time(ev1) / nsteps
            if pg is not None:
                t = torch.tensor([ms], device="cpu" if shared else dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms = float(t.item())
            return ms, L

        _, L = timed_e2e(2, L)             # warm the copy streams
        ms_e2e, L = timed_e2e(max(3, args.steps), L)      # steady state: fill and drain amortised
        bi = x_dev[0].numel() * x_dev[0].element_size()
        bo = out.numel() * out.element_size()
        e2e = {"value": ms_e2e if shape.name != "C2" else G * T / (ms_e2e / 1e3), "unit": "ms" if shape.name != "C2" else "tokens/s",
               "h2d_bytes_per_step": bi * world, "d2h_bytes_per_step": bo * world,
               "pipelined": "H2D(L+1) and D2H(L) on copy streams overlap compute(L+1); double-buffered x/out"}
    rt.check()
    # ---- roofline: the dominant kernel is grouped GEMM1 (4HF FLOPs per routed pair).  Its
    #      algorithmic bytes are the weights of every active (expert, rank) slot + the rows
    #      read and the activations written; the bound is whichever roof is higher.
    pairs = G * T * shape.k
    fl1 = 4.0 * H * shape.F * pairs / world
    fl2 = 2.0 * H * shape.F * pairs / world
    active = int((sp.sum(axis=0) > 0).sum())            # (expert, dest) slots with rows
    by1 = (active * 2 * shape.F * H * 2 + pairs * (H * 2 + shape.F * 2)) / world
    by2 = (active * H * shape.F * 2 + pairs * (shape.F * 2 + H * 2)) / world     # Y is fp16 (D2)
    t1 = phases["gemm1"] / 1e3
    t2 = phases["gemm2"] / 1e3
    peak_tf = pk["bf16_tflops_sustained"]
    peak_bw = pk["hbm_gbs"]
    hbm_bound = by1 / (peak_bw * 1e9) > fl1 / (peak_tf * 1e12)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "gemm1_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        if tj.get("config") == shape.name:
            traffic = tj.get("dram_bytes_per_launch")
    # the library runs the expert GEMMs on CTA pairs when T·k·G ≥ 256·E (256-row tiles fill)
    kname = ("grouped_gemm_2cta_kernel<256,6,4,224> (expert GEMM1 + SwiGLU, tcgen05 cta_group::2)"
             if T * shape.k * G >= 256 * shape.E else
             "grouped_gemm_kernel<256,4,4,1,216> (expert GEMM1 + SwiGLU, tcgen05, 1-CTA 128-row tiles)")
    if hbm_bound:
        roof = {"kernel": kname, "bound": "hbm",
                "achieved": by1 / t1 / 1e9, "peak": peak_bw, "unit": "GB/s", "frac": by1 / t1 / 1e9 / peak_bw,
                "traffic": traffic, "peak_kind": f"{pk_kind} hbm_gbs", "algorithmic_bytes_per_launch": by1,
                "gemm2": {"achieved": by2 / t2 / 1e9, "frac": by2 / t2 / 1e9 / peak_bw},
                "tensor_frac": fl1 / t1 / 1e12 / peak_tf}
    else:
        roof = {"kernel": kname, "bound": "tensor",
                "achieved": fl1 / t1 / 1e12, "peak": peak_tf, "unit": "TFLOP/s", "frac": fl1 / t1 / 1e12 / peak_tf,
                "traffic": traffic, "peak_kind": f"{pk_kind} bf16_tflops_sustained",
                "algorithmic_flops_per_launch": fl1, "algorithmic_bytes_per_launch": by1,
                "gemm2": {"achieved": fl2 / t2 / 1e12, "frac": fl2 / t2 / 1e12 / peak_tf},
                "expert_ffn": {"achieved": (fl1 + fl2) / (t1 + t2) / 1e12,
                               "frac": (fl1 + fl2) / (t1 + t2) / 1e12 / peak_tf}}
    # ---- dispatch / combine against the HBM roofline (one GPU: every "peer" store is local HBM)
    if cfg.dedup_wire:   # x read + one row per unique (token, dest) + 16-B meta per slot; Y read + partials out/in + out
        # (wire rows are this process's own ranks' rows; G·T and pairs cover the EP group)
        byd = (G * T * H * 2 + pairs * 16) / world + wire["rows_unique_token_dest"] * H * 2
        byc = (pairs * H * 2 + G * T * H * out.element_size()) / world + 2 * wire["rows_unique_token_dest"] * H * 2
    else:                # x read + one row per routed pair; fp16 Y rows in, bf16/fp32 out
        byd = (G * T * H * 2 + pairs * H * 2) / world
        byc = (pairs * H * 2 + G * T * H * out.element_size()) / world
    # §8(d)'s unit for the All-to-All: 2H bytes per unique (token, REMOTE destination) — the
    # bytes that would cross NVLink on 8 GPUs; here every "remote" row lands in local HBM
    s8d = 2.0 * H * wire["rows_unique_remote"]          # this process's ranks' rows
    disp_ms = phases["dispatch"]
    comb_ms = phases["combine"] + phases["reduce"]
    bw_report = {"dispatch": {"algorithmic_bytes": byd, "GBps": byd / (disp_ms / 1e3) / 1e9,
                              "frac_hbm": byd / (disp_ms / 1e3) / 1e9 / peak_bw,
                              "s8d_bytes": s8d, "s8d_GBps": s8d / (disp_ms / 1e3) / 1e9,
                              "s8d_frac_hbm": s8d / (disp_ms / 1e3) / 1e9 / peak_bw},
                 "combine": {"algorithmic_bytes": byc, "GBps": byc / (comb_ms / 1e3) / 1e9,
                             "frac_hbm": byc / (comb_ms / 1e3) / 1e9 / peak_bw,
                             "s8d_bytes": s8d, "s8d_GBps": s8d / (comb_ms / 1e3) / 1e9},
                 "note": "algorithmic_bytes = this kernel's own HBM traffic model (per-slot rows: x read + 2H per "
                         "routed pair written); s8d = SURVEY §8(d)'s 2H B per unique (token, remote destination). "
                         "One GPU: the 'NVLink' bytes are local HBM, so fractions are of HBM"}
    result = None
    decode = shape.name == "C2"
    if rank == 0 and light:
        rt.close()
        val = (lambda m: G * T / (m / 1e3)) if decode else (lambda m: m)
        return {"metric": METRIC_DECODE if decode else METRIC_PREFILL, "value": val(ms),
                "unit": "tokens/s" if decode else "ms", "ms_per_step": ms, "higher_is_better": decode,
                "config": {"workload": f"{shape.name}: E={shape.E} top-{shape.k} H={H} F={shape.F} "
                                       f"T={T}/rank{' (decode batch)' if decode else ''} EP={G} "
                                       f"({GL} logical ranks per GPU)",
                           "zipf_s": args.zipf, "window_ns": gemm_ns, "n_sat": n_sat,
                           "dedup_wire": bool(cfg.dedup_wire), "out_dtype": "bf16" if args.out_bf16 else "fp32",
                           "gate_fused_predictor": bool(cfg.fuse_gate_predictor)},
                "static_ep": {"value": val(ms_static), "unit": "tokens/s" if decode else "ms",
                              "ms_per_step": ms_static, "speedup_probe_vs_static": ms_static / ms,
                              "phases_ms": static_phases},
                "phases_ms": phases, "gpu_launches": launches, "clocks": clocks, "prefetch": prefetch, "wire": wire,
                "predispatch": pred_disp, "window": window_rep, "bandwidth": bw_report,
                "balance": {"ir_pre": ir_pre, "ir_post": ir_post, "replicas": nrep,
                            "planner_iterations": stats[0]}}
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:      # the oracle baseline: rank 0 at N = 1 only
            inp = oracle_inputs_cpu(shape, args.zipf)
            cpu = cpu_baseline(inp, (alpha_ps, beta_ps, n_sat, bw_Bpus, gemm_ns), args.cpu_tokens)
            del inp
        value = G * T / (ms / 1e3) if decode else ms
        result = {
            "metric": METRIC_DECODE if decode else METRIC_PREFILL,
            "value": value, "unit": "tokens/s" if decode else "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": decode, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic: Hadamard-encoded exact routing, Zipf(s) popularity, hotspots "
                                     "migrating layer to layer, encoded predictor accuracy 0.9; random-init experts",
            "config": {"workload": f"{shape.name}: E={shape.E} top-{shape.k} H={H} F={shape.F} "
                                   f"T={T}/rank EP={G} ({GL} logical ranks per GPU)",
                       "out_dtype": "bf16" if args.out_bf16 else "fp32",
                       "wire": "dedup (one row per unique (token, dest))" if cfg.dedup_wire else "per-slot rows",
                       "gate_fused_predictor": bool(cfg.fuse_gate_predictor),
                       "zipf_s": args.zipf, "replica_budget": 3, "kmax": 16, "alpha_ps": alpha_ps,
                       "beta_ps": beta_ps, "n_sat": n_sat, "window_ns": gemm_ns,
                       "l2": "inputs larger than L2 (x 268 MB/layer at C1, weights 1.2 GB/parity); no flush"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "phases_ms": phases,
            "static_ep": {"ms_per_step": ms_static, "speedup_probe_vs_static": ms_static / ms,
                          "phases_ms": static_phases},
            "ep_emulation": ep_em,
            "balance": {"ir_pre": ir_pre, "ir_post": ir_post, "replicas": nrep,
                        "planner": {"iterations": stats[0], "transfers": stats[1], "maxL_before_ps": stats[2],
                                    "maxL_after_ps": stats[3]},
                        "predicted_load_fidelity": load_fidelity},
            "bandwidth": bw_report,
            "wire": wire,
            "window": window_rep,
            "prefetch": prefetch,
            "setup_s": gen_s,
        }
    rt.close()
    return result


# =============================================================================
# oracle (CPU) — cpu_baseline leg and --impl reference arm
# =============================================================================

class OracleInputs:
    """fp64 host copies of one layer's full-size inputs (untimed setup): x of every rank,
    the router of this layer and of the next (predictor prior), the predictor residual, and
    the expert weights (decoded on first use and kept while they fit a host budget)."""

    def __init__(self, shape, x, W, Wn, r1, r2, w13, w2, budget_bytes=24 << 30):
        f = pi.bf16_to_numpy_f64
        self.sh = shape
        self.xs = [f(x[r]) for r in range(x.shape[0])]
        self.W, self.Wn = f(W), f(Wn)
        self.r1, self.r2 = f(r1), f(r2)
        self.w13, self.w2 = w13, w2          # bf16 tensors [E, 2F, H] / [E, H, F] (any device)
        self.cache_ok = 8 * 3 * shape.H * shape.F * shape.E <= budget_bytes
        self._c13, self._c2 = {}, {}
        if self.cache_ok:                    # decode every expert now (untimed)
            for e in range(shape.E):
                self.expert(e)

    def expert(self, e):
        if e in self._c13:
            return self._c13[e], self._c2[e]
        f = pi.bf16_to_numpy_f64
        a, b = f(self.w13[e]), f(self.w2[e])
        if self.cache_ok:
            self._c13[e], self._c2[e] = a, b
        return a, b


class _Experts:
    def __init__(self, inp, which):
        self.inp, self.which = inp, which

    def __getitem__(self, e):
        return self.inp.expert(e)[self.which]


def oracle_inputs_cpu(shape, zipf, layer=1):
    """The reference arm's inputs, generated on the host with the probe arm's generator."""
    li = pi.layer_inputs(shape, 0, layer, zipf, wrap=POOL)
    w13, w2 = pi.expert_weights(shape, layer % 2)
    r1, r2 = pi.predictor_residual(shape, (layer + 1) % 2)
    return OracleInputs(shape, li.x, pi.router_weight(shape, layer % 2), pi.router_weight(shape, (layer + 1) % 2),
                        r1, r2, w13, w2)


def oracle_layer_measured(inp: OracleInputs, sample_tokens, consts):
    """One step of the fp64 oracle over the whole hot path of one layer (§8(a) a1-a8).

    MEASURED at full size: gate (a1) and predictor (a2) over every token of every rank, the
    planner (a4) on the full n̂, materialize + dispatch layout (a5, a6) over every routed pair.
    MEASURED on a sample: the expert FFN + combine (a7, a8) for `sample_tokens` tokens of every
    rank (their cost is exactly per token: each (token, slot) is one fp64 SwiGLU), composed
    to the full layer as t_ffn · T / sample.  Returns (composed_ms, step_ms, parts)."""
    import oracle as O
    sh = inp.sh
    G, E, k, T = sh.G, sh.E, sh.k, sh.T
    alpha_ps, beta_ps, n_sat, bw, win = consts
    parts = {}
    t0 = time.perf_counter()
    gates = [O.gate(inp.xs[s], inp.W, None, k) for s in range(G)]
    t1 = time.perf_counter()
    nhat = np.stack([O.predict_counts(inp.xs[s], inp.Wn, None, inp.r1, inp.r2, k)[0] for s in range(G)])
    t2 = time.perf_counter()
    pcfg = O.PlannerConfig(G=G, E=E, replica_budget=3, kmax=16, alpha_ps=alpha_ps, beta_ps=beta_ps, n_sat=n_sat,
                           bw_bytes_per_us=bw, expert_bytes=6 * sh.H * sh.F)
    plan = O.plan_greedy(nhat, [win] * G, pcfg)
    t3 = time.perf_counter()
    ids = [g[0] for g in gates]
    n = np.stack([g[2] for g in gates])
    split = O.materialize(n, plan.quota, plan.replicas, G, E)
    O.dispatch_layout(ids, split, plan.replicas, G, E)
    t4 = time.perf_counter()
    ns = min(sample_tokens, T)
    toks = [list(range(ns))] * G
    O.moe_outputs_ranks(inp.xs, ids, [g[1] for g in gates], _Experts(inp, 0), _Experts(inp, 1), toks)
    t5 = time.perf_counter()
    parts = {"gate_ms": (t1 - t0) * 1e3, "predictor_ms": (t2 - t1) * 1e3, "planner_ms": (t3 - t2) * 1e3,
             "materialize_layout_ms": (t4 - t3) * 1e3, "experts_combine_sample_ms": (t5 - t4) * 1e3,
             "experts_combine_full_ms": (t5 - t4) * 1e3 * T / ns}
    composed = (t4 - t0) * 1e3 + parts["experts_combine_full_ms"]
    return composed, (t5 - t0) * 1e3, parts


def oracle_sample_note(shape, ns, inp):
    return (f"gate + predictor over all {shape.G}x{shape.T} tokens, planner on the full n̂, materialize + "
            f"layout over all pairs: measured; fp64 SwiGLU experts + combine measured on {ns} tokens/rank "
            f"and composed x{shape.T // ns} (exact per-token cost); expert weights "
            f"{'pre-decoded (untimed)' if inp.cache_ok else 'decoded inside the timed region'}")


def cpu_baseline(inp, consts, sample_tokens):
    composed, step_ms, parts = oracle_layer_measured(inp, sample_tokens, consts)
    shape = inp.sh
    decode = shape.name == "C2"
    full = shape.G * shape.T
    return {"value": full / (composed / 1e3) if decode else composed, "unit": "tokens/s" if decode else "ms",
            "cores": _cores(), "kind": "oracle", "sample": oracle_sample_note(shape, min(sample_tokens, shape.T), inp),
            "measured_step_ms": step_ms, "parts_ms": parts}


def _cores():
    try:
        import threadpoolctl
        n = [p.get("num_threads") for p in threadpoolctl.threadpool_info() if p.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    shape = pi.SHAPES[args.config]
    t_setup = time.time()
    inp = oracle_inputs_cpu(shape, args.zipf)
    from paper_2602_00509_b200.costs import cost_model as cm, peaks as pks, window_ns as wn
    pk, _ = pks()
    a, b, nsat, bw = cm(shape.H, shape.F, pk)
    consts = (a, b, nsat, bw, wn(shape.H, shape.F, shape.T, shape.k, pk, E=shape.E, G=shape.G))
    setup_s = time.time() - t_setup
    ns = args.cpu_tokens
    for _ in range(args.warmup):
        oracle_layer_measured(inp, ns, consts)
    comp, steps_ms, parts_all = [], [], []
    t_run = time.time()
    for _ in range(args.steps):
        c, sm, parts = oracle_layer_measured(inp, ns, consts)
        comp.append(c)
        steps_ms.append(sm)
        parts_all.append(parts)
    run_s = time.time() - t_run
    ms = statistics.mean(comp)
    decode = shape.name == "C2"
    full = shape.G * shape.T
    value = full / (ms / 1e3) if decode else ms
    unit = "tokens/s" if decode else "ms"
    step_ms = statistics.mean(steps_ms)
    parts = {k: statistics.mean(p[k] for p in parts_all) for k in parts_all[0]}
    note = oracle_sample_note(shape, min(ns, shape.T), inp)
    out = {"impl": "reference", "metric": METRIC_DECODE if decode else METRIC_PREFILL, "value": value,
           "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": step_ms, "composed_layer_ms": ms,
           "higher_is_better": decode, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same generator as the probe arm)",
           "config": {"workload": f"{shape.name}: E={shape.E} top-{shape.k} H={shape.H} F={shape.F} "
                                  f"T={shape.T}/rank EP={shape.G} (fp64 oracle on the host, all ranks in one process)",
                      "sample": note},
           "cpu_baseline": {"value": value, "unit": unit, "kind": "oracle", "cores": _cores(), "sample": note,
                            "parts_ms": parts},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "timing": {"ms_per_step": "measured wall time of one sampled oracle step",
                      "value": "composed full-layer time (measured full-size stages + per-token expert cost x T)",
                      "timed_run_s": run_s, "setup_s": setup_s,
                      "fits_in_driver_run": bool(step_ms * args.steps / 1e3 <= run_s * 1.05)}}
    print(json.dumps(out), flush=True)
    return out


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="probe", choices=["probe", "reference"])
    ap.add_argument("--config", default="C1", choices=["C1", "C2", "C3"])
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-emulation", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the C2 decode sub-measurement of the C1 line")
    ap.add_argument("--wire", default="auto", choices=["auto", "slot", "dedup"],
                    help="dispatch/combine wire format (auto: dedup across processes, per-slot in one process)")
    ap.add_argument("--modeled-window", action="store_true",
                    help="plan with the modeled hiding window instead of the measured one (R26)")
    ap.add_argument("--attn-ns", type=int, default=0, help="attention window added to the measured GEMM window")
    ap.add_argument("--no-dedup-sub", action="store_true", help="skip the dedup-wire sub-measurement")
    ap.add_argument("--ep", type=int, default=0, help="EP size G (default: the config's, 8)")
    ap.add_argument("--out-bf16", action="store_true", help="bf16 layer output instead of fp32 (the parity-tested default)")
    ap.add_argument("--cap", type=float, default=4.0, help="receive capacity per rank in units of T·k")
    ap.add_argument("--aux-sms", type=int, default=0, help="grid cap of the aux-stream predictor GEMMs (0: #SMs/2)")
    ap.add_argument("--aux-start", type=int, default=0, help="1: predictor starts after dispatch (not beside it)")
    ap.add_argument("--pred-maxreg", type=int, default=0, help="192: register-capped predictor GEMMs")
    ap.add_argument("--pred-pair", type=int, default=None, choices=[0, 1],
                    help="predictor Ŵ1·x GEMM on CTA pairs (library default 1)")
    ap.add_argument("--l2hint", type=lambda v: int(v, 0), default=0, help="expert-GEMM TMA L2 hint mask (probe.h)")
    ap.add_argument("--cpu-tokens", type=int, default=1024, help="oracle expert-FFN sample, tokens per rank")
    ap.add_argument("--epi-topk", type=int, default=0, help="1: router/predictor top-k in the GEMM epilogue")
    ap.add_argument("--gate-fuse", default="auto", choices=["auto", "0", "1"],
                    help="gate GEMM also computes the next layer's prior + predictor activation "
                         "(auto: when several logical ranks share the GPU)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    return args


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_probe(args)


if __name__ == "__main__":
    main()

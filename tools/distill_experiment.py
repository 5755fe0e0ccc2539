"""Streaming distillation experiment (P:573 / P:586 fidelity metrics).

A stream of synthetic batches with a fixed "feature drift" between the predictor's input
and the teacher's input (probe_inputs.distill_task: the drift relabels the routing mass of
drift_frac·E experts).  The residual starts at Ŵ² = 0 (the "untrained" predictor = frozen
router only), is trained by probe_distill_grad/apply on each batch, and the three
fidelity metrics are measured on a held-out batch every `--every` steps.  Also times one
distillation step (CUDA events).  Prints JSON lines.

  python tools/distill_experiment.py --config C1 --tokens 2048 --steps 300 --lr 8
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import probe_inputs as pi  # noqa: E402
from paper_2602_00509_b200 import ProbeConfig, ProbeRuntime  # noqa: E402
from paper_2602_00509_b200._lib import OPT_AUX_SMS  # noqa: E402
from paper_2602_00509_b200.distill import PredictorDistiller, metrics  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--tokens", type=int, default=2048, help="tokens per rank per batch")
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--lr", type=float, nargs="+", default=[8.0])
    ap.add_argument("--drift", type=float, default=0.35)
    ap.add_argument("--zipf", type=float, default=1.2)
    ap.add_argument("--w1-scale", type=float, default=1.0)
    ap.add_argument("--sms", type=int, default=0, help="grid cap of the distillation GEMMs (0: default #SMs/2)")
    a = ap.parse_args()
    sh = pi.SHAPES[a.config].with_(T=a.tokens)
    torch.cuda.init()
    train = [pi.distill_task(sh, s, zipf_s=a.zipf, drift_frac=a.drift, device="cuda") for s in range(a.batches)]
    held = pi.distill_task(sh, 1000, zipf_s=a.zipf, drift_frac=a.drift, device="cuda")
    W = held.W
    N = sh.G * sh.T
    for lr in a.lr:
        rt = ProbeRuntime(ProbeConfig(G=sh.G, E=sh.E, k=sh.k, H=sh.H, F=64, T=sh.T, h=sh.h))
        if a.sms:
            rt.set_option(OPT_AUX_SMS, a.sms)
        g = pi.torch_gen(sh.name, "distill-init")
        w1 = (torch.randn(sh.h, sh.H, generator=g) * a.w1_scale / math.sqrt(sh.H)).to(torch.bfloat16).cuda()
        w2 = torch.zeros(sh.E, sh.h, dtype=torch.bfloat16, device="cuda")
        d = PredictorDistiller(rt, w1, w2)

        def evaluate():
            d.grad(held.x, held.x_next, W)
            return metrics(d.stats, N, sh.k)

        hist = [dict(step=0, **evaluate())]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for s in range(1, a.steps + 1):
            b = train[(s - 1) % len(train)]
            t0.record()
            d.step(b.x, b.x_next, W, lr=lr, want_metrics=False)
            t1.record()
            if s % a.every == 0 or s == a.steps:
                torch.cuda.synchronize()
                ms.append(t0.elapsed_time(t1))
                hist.append(dict(step=s, **evaluate()))
        print(json.dumps({"config": a.config, "tokens_per_batch": N, "lr": lr, "drift_frac": a.drift,
                          "zipf_s": a.zipf, "E": sh.E, "k": sh.k, "H": sh.H, "h": sh.h,
                          "untrained": hist[0], "distilled": hist[-1], "history": hist,
                          "ms_per_step_sampled": ms}))
        rt.close()


if __name__ == "__main__":
    main()

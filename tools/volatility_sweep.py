"""BASELINE.json configs[4] — volatility sweep: C1 (prefill) and C2 (decode) shapes ×
Zipf s ∈ {0.5, 0.75, 1.0, 1.25, 1.5} × EP size G ∈ {1, 2, 4, 8}, hotspots re-permuted every
layer, PROBE vs static EP.  One B200: the whole EP group runs on the GPU (G logical ranks);
the straggler effect of Eq. 3 is reproduced by the EP emulation (expert GEMMs split into G
CTA sets), whose static-EP and PROBE times are the comparison.  Each point is one
`bench.run_probe` call (same timing method as bench.py).

    python tools/volatility_sweep.py [--shapes C1,C2] [--steps 10] [--out profiles/volatility_r01.jsonl]
"""
import argparse
import io
import json
import os
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def point(shape, s, G, steps):
    argv = ["--steps", str(steps), "--warmup", "3", "--config", shape, "--zipf", str(s), "--ep", str(G),
            "--no-e2e", "--no-cpu", "--no-decode", "--no-dedup-sub"] + (["--no-emulation"] if G == 1 else [])
    a = bench.parse_args(argv)
    with redirect_stdout(io.StringIO()):
        r = bench.run_probe(a)
    em = r.get("ep_emulation") or {}
    b = r["balance"]
    return {"shape": shape, "zipf_s": s, "G": G, "metric": r["metric"], "unit": r["unit"], "probe": r["value"],
            "static_ep_ms": r["static_ep"]["ms_per_step"], "probe_ms": r["ms_per_step"],
            "em_static_ms": em.get("static_ep_ms"), "em_probe_ms": em.get("probe_ms"),
            "em_speedup": em.get("speedup_probe_vs_static"), "ir_pre": b["ir_pre"], "ir_post": b["ir_post"],
            "replicas": b["replicas"], "planner_iters": b["planner"]["iterations"],
            "pred_fidelity": b["predicted_load_fidelity"], "wait_ms": r["phases_ms"]["wait"],
            "prefetch_part1_MB": r["prefetch"]["part1_MB_per_layer"], "prefetch_part2_MB": r["prefetch"]["part2_MB_per_layer"],
            "clocks": r["clocks"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="C1,C2")
    ap.add_argument("--zipf", default="0.5,0.75,1.0,1.25,1.5")
    ap.add_argument("--eps", default="8,4,2,1")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "volatility_r01.jsonl"))
    args = ap.parse_args()
    with open(args.out, "w") as f:
        for shape in args.shapes.split(","):
            for G in [int(g) for g in args.eps.split(",")]:
                for s in [float(z) for z in args.zipf.split(",")]:
                    p = point(shape, s, G, args.steps)
                    f.write(json.dumps(p) + "\n")
                    f.flush()
                    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()
                                      if k != "clocks"}), flush=True)


if __name__ == "__main__":
    main()

"""Debug aid: repeat the C2 full-size layer on the GPU and report which outputs disagree with the oracle."""
import dataclasses
import os
import sys

import numpy as np

sys.path[:0] = [".", "tests"]
import probe_inputs as pi
from layer_harness import run_gpu, run_oracle
from test_gpu_fullsize import bench_case

base = bench_case(pi.C2, sample=32)
orc = None
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["default", "sync", "b0"]
for it in range(int(os.environ.get("REPS", "3"))):
    for mode in modes:
        case = dataclasses.replace(base, replica_budget=0) if mode == "b0" else base
        if mode == "sync":
            os.environ["PROBE_TEST_SYNC_L0"] = "1"
        else:
            os.environ.pop("PROBE_TEST_SYNC_L0", None)
        gpu, inputs = run_gpu(case)
        if orc is None or mode == "b0" or orc[0] != (mode == "b0"):
            import pickle
            cache = f"/tmp/c2dbg_orc_{mode == 'b0'}.pkl"
            if os.path.exists(cache):
                orc = pickle.load(open(cache, "rb"))
            else:
                orc = (mode == "b0", run_oracle(case, inputs))
                pickle.dump(orc, open(cache, "wb"))
        o = orc[1]
        ref = o["ref"][0]
        toks = o["tokens"]
        rms = np.sqrt(np.mean(np.concatenate([q.reshape(-1) for q in ref["out"]]) ** 2))
        nbad = 0
        for r in range(case.shape.G):
            err = np.abs(gpu["out"][0][r][toks[r]] - ref["out"][r])
            bad = np.argwhere(err > 0.02 * rms)
            if len(bad):
                nbad += len(bad)
                tb = sorted(set(toks[r][i] for i in bad[:, 0]))
                cols = sorted(set(bad[:, 1].tolist()))
                print(f"  {mode} it{it} rank {r}: {len(bad)} bad, tokens {tb[:8]}, cols {cols[:6]}..{cols[-3:]} "
                      f"({len(cols)} cols), ids {gpu['ids'][0][r][tb[0]].tolist()}, max {err.max() / rms:.2f} RMS", flush=True)
        print(mode, "it", it, "bad", nbad, "replicas", int((gpu["replicas"] >= 0).sum()), flush=True)

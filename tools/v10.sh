mkdir -p gpurun_out
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  PROBE_Y_WIDE=1 timeout 600 python bench.py $Q > gpurun_out/v10_w1_$i.json 2>&1
  PROBE_Y_WIDE=0 timeout 600 python bench.py $Q > gpurun_out/v10_w0_$i.json 2>&1
done
PROBE_Y_WIDE=1 timeout 600 python bench.py $Q --config C2 > gpurun_out/v10_c2_w1.json 2>&1
PROBE_Y_WIDE=0 timeout 600 python bench.py $Q --config C2 > gpurun_out/v10_c2_w0.json 2>&1
for f in gpurun_out/v10_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["ms_per_step"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if k in ("gate","dispatch","gemm1","gemm2","combine")), "| static g2", round(sp["gemm2"],3), d["clocks"]["sm_mhz"])
PY
done

mkdir -p gpurun_out
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for g in 0 1; do
  timeout 600 python bench.py $Q --config C2 --gate-fuse $g > gpurun_out/v7_c2_g$g.json 2>&1
  timeout 900 python bench.py $Q --config C3 --steps 5 --warmup 3 --cap 3 --gate-fuse $g > gpurun_out/v7_c3_g$g.json 2>&1
done
for f in gpurun_out/v7_c*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["value"],3), round(d["static_ep"]["value"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if v > 0.004), "| static gate", round(sp["gate"],3), "disp", round(sp["dispatch"],3), d["clocks"]["sm_mhz"], d["prefetch"]["part1_MB_per_layer"], d["prefetch"]["part2_MB_per_layer"])
PY
done

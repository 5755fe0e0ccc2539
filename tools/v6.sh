mkdir -p gpurun_out
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  timeout 600 python bench.py $Q --gate-fuse 0 > gpurun_out/v6_c1_g0_$i.json 2>&1
  timeout 600 python bench.py $Q --gate-fuse 1 > gpurun_out/v6_c1_g1_$i.json 2>&1
done
for f in gpurun_out/v6_c1_g*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["value"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if v > 0.004), "| static gate", round(sp["gate"],3), "disp", round(sp["dispatch"],3), "total", round(sp["total"],3), d["clocks"]["sm_mhz"])
PY
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_" -c 60 --csv \
    --log-file gpurun_out/v6_launches_g1.csv python bench.py --steps 2 --warmup 3 $Q --gate-fuse 1 > /dev/null 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -s > gpurun_out/v6_tests.log 2>&1
tail -3 gpurun_out/v6_tests.log

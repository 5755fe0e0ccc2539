mkdir -p gpurun_out
python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py -m gpu -q -p no:cacheprovider --timeout 600 -k "topk or epilogue or C0" -rf --tb=short > gpurun_out/v8_tests.log 2>&1
tail -2 gpurun_out/v8_tests.log
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  timeout 600 python bench.py $Q --gate-fuse 0 --epi-topk 0 > gpurun_out/v8_e0_$i.json 2>&1
  timeout 600 python bench.py $Q --gate-fuse 0 --epi-topk 1 > gpurun_out/v8_e1_$i.json 2>&1
  timeout 600 python bench.py $Q --gate-fuse 1 --epi-topk 1 > gpurun_out/v8_g1e1_$i.json 2>&1
done
for f in gpurun_out/v8_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["ms_per_step"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if v > 0.004 and k in ("gate","select","dispatch","gemm1","gemm2","total")), "| static gate", round(sp["gate"],3), "sel", round(sp["select"],3), "disp", round(sp["dispatch"],3), d["clocks"]["sm_mhz"])
PY
done

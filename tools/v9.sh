mkdir -p gpurun_out
for i in 1 2; do
  PROBE_Y_WIDE=1 python tools/gemm_ab.py | tail -1
  PROBE_Y_WIDE=0 python tools/gemm_ab.py | tail -1
done
python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py -m gpu -q -p no:cacheprovider --timeout 600 -k "C0 or ragged or C2 or pair or fp16" -rf --tb=short > gpurun_out/v9_tests.log 2>&1
tail -2 gpurun_out/v9_tests.log
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  PROBE_Y_WIDE=1 timeout 600 python bench.py $Q > gpurun_out/v9_w1_$i.json 2>&1
  PROBE_Y_WIDE=0 timeout 600 python bench.py $Q > gpurun_out/v9_w0_$i.json 2>&1
done
for f in gpurun_out/v9_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["ms_per_step"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if k in ("gate","dispatch","gemm1","gemm2","combine")), "| static g2", round(sp["gemm2"],3), "gemm2 frac", round(d["roofline"]["gemm2"]["frac"],3), d["clocks"]["sm_mhz"])
PY
done

mkdir -p gpurun_out
for i in 1 2; do
  PROBE_L2PF=74 python tools/gemm_ab.py | tail -1
  PROBE_L2PF=0 python tools/gemm_ab.py | tail -1
done
PROBE_L2PF=37 python tools/gemm_ab.py | tail -1
PROBE_L2PF=148 python tools/gemm_ab.py | tail -1
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  PROBE_L2PF=74 timeout 600 python bench.py $Q > gpurun_out/v11_p1_$i.json 2>&1
  PROBE_L2PF=0 timeout 600 python bench.py $Q > gpurun_out/v11_p0_$i.json 2>&1
done
for f in gpurun_out/v11_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["ms_per_step"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      " ".join(f"{k} {v:.3f}" for k,v in ph.items() if k in ("gate","dispatch","gemm1","gemm2","combine")), "| static g1", round(sp["gemm1"],3), "g2", round(sp["gemm2"],3), d["clocks"]["sm_mhz"])
PY
done
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider -k "pair or f16 or multi_tile" --tb=line 2>&1 | tail -2

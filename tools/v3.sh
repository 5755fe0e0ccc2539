mkdir -p gpurun_out
for i in 1 2; do
  python tools/gemm_ab.py 2>&1 | tail -1
  PROBE_LIB_PATH=$PWD/paper_2602_00509_b200/libprobe_old.so python tools/gemm_ab.py 2>&1 | tail -1
done
python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider --timeout 600 -k "gate or natural" -rf --tb=short -s > gpurun_out/v3_layer.log 2>&1
tail -3 gpurun_out/v3_layer.log; grep "natural\|gate" gpurun_out/v3_layer.log | head -20
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  timeout 600 python bench.py $Q --gate-fuse 0 > gpurun_out/v3_c1_g0_$i.json 2>&1
  timeout 600 python bench.py $Q --gate-fuse 1 > gpurun_out/v3_c1_g1_$i.json 2>&1
done
for f in gpurun_out/v3_c1_g*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["value"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      "gate", round(ph["gate"],3), "sel", round(ph["select"],3), "disp", round(ph["dispatch"],3), "g1", round(ph["gemm1"],3), "g2", round(ph["gemm2"],3), "static disp", round(sp["dispatch"],3), "g1", round(sp["gemm1"],3), "g2", round(sp["gemm2"],3), d["clocks"]["sm_mhz"])
PY
done

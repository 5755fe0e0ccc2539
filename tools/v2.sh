mkdir -p gpurun_out
# GEMM A/B: producer one tile ahead (in-tree) vs the previous build
for i in 1 2; do
  python tools/gemm_ab.py > gpurun_out/v2_gemm_new_$i.json 2>&1; cat gpurun_out/v2_gemm_new_$i.json | tail -1
  PROBE_LIB_PATH=$PWD/paper_2602_00509_b200/libprobe_old.so python tools/gemm_ab.py > gpurun_out/v2_gemm_old_$i.json 2>&1; tail -1 gpurun_out/v2_gemm_old_$i.json
done
# fused gate + predictor stage 1: parity cases, full-size bench configuration, A/B timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider --timeout 600 -k "gate_fused or gate-fused or C0 or relabel" -rf --tb=short > gpurun_out/v2_layer.log 2>&1
tail -3 gpurun_out/v2_layer.log
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider --timeout 900 -k "C1-bench or C2 or C3" -rf --tb=short -s > gpurun_out/v2_full.log 2>&1
tail -3 gpurun_out/v2_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1; tail -2 gpurun_out/v2_smoke.log
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
for i in 1 2; do
  timeout 600 python bench.py $Q --gate-fuse 0 > gpurun_out/v2_c1_g0_$i.json 2>&1
  timeout 600 python bench.py $Q --gate-fuse 1 > gpurun_out/v2_c1_g1_$i.json 2>&1
done
for f in gpurun_out/v2_c1_g*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph=d["phases_ms"]; sp=d["static_ep"]["phases_ms"]
print(sys.argv[1], round(d["value"],3), round(d["static_ep"]["ms_per_step"],3), round(d["static_ep"]["speedup_probe_vs_static"],3),
      "gate", round(ph["gate"],3), "sel", round(ph["select"],3), "disp", round(ph["dispatch"],3), "static disp", round(sp["dispatch"],3), d["clocks"]["sm_mhz"])
PY
done
timeout 300 python bench.py $Q --config C2 > gpurun_out/v2_c2.json 2>&1; tail -c 300 gpurun_out/v2_c2.json

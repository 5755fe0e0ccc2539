mkdir -p gpurun_out
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub --steps 10"
timeout 300 python bench.py $Q > gpurun_out/g2_base.json 2>&1
PROBE_DEBUG_GEMM2_REPEAT=1 timeout 300 python bench.py $Q > gpurun_out/g2_rep.json 2>&1
PROBE_DEBUG_GAP_US=300 timeout 300 python bench.py $Q > gpurun_out/g2_gap.json 2>&1
PROBE_DEBUG_GAP_US=1000 timeout 300 python bench.py $Q > gpurun_out/g2_gap1000.json 2>&1

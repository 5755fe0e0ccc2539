mkdir -p gpurun_out
python tools/gemm2_groups.py > gpurun_out/gemm2_groups.json 2>&1

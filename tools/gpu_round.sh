mkdir -p gpurun_out
python tools/gemm_stats.py 6 > gpurun_out/gemm_stats2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_select|grouped_gemm" -s 14 -c 5 \
    -o gpurun_out/full_aux_r02 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub > gpurun_out/ncu_aux.log 2>&1

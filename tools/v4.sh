mkdir -p gpurun_out
python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider --timeout 600 -k "natural or gate" -rf --tb=short -s > gpurun_out/v4_layer.log 2>&1
tail -3 gpurun_out/v4_layer.log
Q="--no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_|sgemm" -c 120 --csv \
    --log-file gpurun_out/v4_launches_g1.csv python bench.py --steps 2 --warmup 3 $Q --gate-fuse 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_2cta" -s 12 -c 3 \
    -o gpurun_out/v4_fused python bench.py --steps 1 --warmup 3 $Q --gate-fuse 1 > gpurun_out/v4_ncu.log 2>&1
tail -2 gpurun_out/v4_ncu.log

mkdir -p gpurun_out
python tools/gemm_stats.py 6 > gpurun_out/gemm_stats3.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -k "gemm or layer_parity or fullsize_parity[C1-bench]" > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
for i in 1 2; do timeout 300 python bench.py $Q > gpurun_out/ab_tma_$i.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_|sgemm" -c 60 --csv \
    --log-file gpurun_out/launches_tma.csv python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1

mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -k "not fullsize" > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -s -k "fullsize_parity[C3 or fullsize_parity[C1-relabel" > gpurun_out/t2.log 2>&1
tail -3 gpurun_out/t2.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
for i in 1 2; do timeout 300 python bench.py $Q > gpurun_out/ab_p2_$i.json 2>&1; timeout 300 python bench.py $Q --pred-pair 0 > gpurun_out/ab_p0_$i.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_select" -c 14 --csv \
    --log-file gpurun_out/launches_p2.csv python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1

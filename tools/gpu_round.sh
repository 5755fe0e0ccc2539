# one gpurun session: GPU tests (layer + predictor + full-size C1), A/B of the predictor on CTA pairs
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -s -k "layer_parity or planner or fullsize_parity[C1-bench] or fullsize_parity[C1-relabel" > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
for i in 1 2; do
  timeout 300 python bench.py $Q > gpurun_out/ab_pair1_$i.json 2>&1
  timeout 300 python bench.py $Q --pred-pair 0 > gpurun_out/ab_pair0_$i.json 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_|sgemm" -c 60 --csv \
    --log-file gpurun_out/launches_pair.csv python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1

# one gpurun session: GPU tests (all but full-size), A/B of the aux-track placement, ncu evidence
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "not fullsize" -rf --tb=short > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
for i in 1 2 3; do
  timeout 300 python bench.py $Q > gpurun_out/ab_default_$i.json 2>&1
  timeout 300 python bench.py $Q --aux-start 1 --aux-sms 37 > gpurun_out/ab_after37_$i.json 2>&1
done
timeout 300 python bench.py $Q --config C2 > gpurun_out/b_c2.json 2>&1
timeout 300 python bench.py $Q --config C2 --modeled-window > gpurun_out/b_c2_modeled.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_2cta|k_dispatch|k_combine" -s 8 -c 8 \
    -o gpurun_out/full_r02 python bench.py --steps 1 --warmup 3 $Q > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dispatch_dedup|k_expand|k_combine_partial|k_combine_reduce|k_predispatch" -s 20 -c 10 \
    -o gpurun_out/full_dedup_r02 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-emulation --no-decode \
    > gpurun_out/ncu_dedup.log 2>&1
ls -la gpurun_out

# final light validation: every GPU test, smoke, the driver's default bench line, reference arm
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -s > gpurun_out/t_all.log 2>&1
tail -3 gpurun_out/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
tail -c 300 gpurun_out/bench_r02.json
timeout 900 python bench.py --impl reference > gpurun_out/ref_r02.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm|k_|sgemm" -c 200 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm|k_dispatch|k_combine|k_select" -s 16 -c 8 \
    -o gpurun_out/full_r02 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-decode --no-dedup-sub --no-emulation > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --no-decode --no-dedup-sub --config C2 > gpurun_out/bench_r02_c2.json 2>&1
timeout 900 python bench.py --no-cpu --no-e2e --no-decode --no-dedup-sub --config C3 --steps 5 --warmup 3 --cap 3 > gpurun_out/bench_r02_c3.json 2>&1

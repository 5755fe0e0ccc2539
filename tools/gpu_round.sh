# one gpurun session: GEMM study (wait counters), GPU tests, bench, 2-process functional bench
mkdir -p gpurun_out
python tools/gemm_stats.py 6 > gpurun_out/gemm_stats.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --tb=short -k "not fullsize" > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
PROBE_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/bench_shared2.json 2> gpurun_out/bench_shared2.err
tail -c 300 gpurun_out/bench_shared2.err

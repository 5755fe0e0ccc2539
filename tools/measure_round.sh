#!/bin/bash
# Round-end measurement batch (run on a B200 box from the repo root): GPU tests, smoke, bench lines
# for C1/C2/C3, the N>1 path on a shared GPU, the ncu launch list and one ncu --set full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/f_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/f_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench_c1.log 2>&1
timeout 400 python bench.py --config C2 > gpurun_out/f_bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --cap 2.5 --steps 5 --no-cpu > gpurun_out/f_bench_c3.log 2>&1
PROBE_BENCH_SHARED_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/f_shared2.log 2>&1; echo exit=$? >> gpurun_out/f_shared2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped|k_" --csv --log-file gpurun_out/ncu_launches_${TAG:-r01c}.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-emulation > gpurun_out/f_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_2cta|k_dispatch|k_combine" -s 12 -c 4 -o gpurun_out/full_${TAG:-r01c} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-emulation > gpurun_out/f_ncu2.log 2>&1

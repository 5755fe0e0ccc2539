mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/v1_smi.txt
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -x -rf --tb=short > gpurun_out/v1_tests.log 2>&1
tail -3 gpurun_out/v1_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1; tail -2 gpurun_out/v1_smoke.log
timeout 900 python bench.py > gpurun_out/v1_bench.json 2> gpurun_out/v1_bench.err
python -c "import json;d=json.load(open('gpurun_out/v1_bench.json'));print(d['value'],d['static_ep']['ms_per_step'],d['roofline']['frac'],d['roofline']['gemm2'])"

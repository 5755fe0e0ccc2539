set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "not fullsize" -rf --tb=short > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider --timeout 1200 -rf --tb=short > gpurun_out/t2.log 2>&1
tail -3 gpurun_out/t2.log

# one gpurun session: GPU tests (all but full-size) + bench variants (outputs in gpurun_out/)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "not fullsize" -rf --tb=short > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
timeout 300 python bench.py $Q > gpurun_out/b_default.json 2> gpurun_out/b_default.err
timeout 300 python bench.py $Q --aux-sms 148 > gpurun_out/b_aux148.json 2>&1
timeout 300 python bench.py $Q --pred-maxreg 192 > gpurun_out/b_r192.json 2>&1
timeout 300 python bench.py $Q --aux-start 1 > gpurun_out/b_after.json 2>&1
timeout 300 python bench.py $Q --aux-sms 37 > gpurun_out/b_aux37.json 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 400 gpurun_out/bench.err

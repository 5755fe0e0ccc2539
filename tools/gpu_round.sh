# one gpurun session: GPU tests (all but full-size) + bench variants (outputs in gpurun_out/)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "not fullsize" -rf --tb=short > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
Q="--no-cpu --no-e2e --no-emulation --no-decode --no-dedup-sub"
timeout 300 python bench.py $Q > gpurun_out/b_default.json 2>&1
timeout 300 python bench.py $Q --aux-start 1 > gpurun_out/b_after.json 2>&1
timeout 300 python bench.py $Q --aux-sms 37 > gpurun_out/b_aux37.json 2>&1
timeout 300 python bench.py $Q --aux-start 1 --aux-sms 37 > gpurun_out/b_after37.json 2>&1
for h in 0x10 0x20 0x30 0x11 0x22 0x33 0x77; do
  timeout 300 python bench.py $Q --l2hint $h > gpurun_out/b_l2_$h.json 2>&1
done
timeout 300 python bench.py $Q --config C2 > gpurun_out/b_c2.json 2>&1
timeout 900 python bench.py $Q --config C3 --steps 5 --warmup 3 --cap 3 > gpurun_out/b_c3.json 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_parity.py -q -x -k "graph or determinism or host" > gpurun_out/pytest45.log 2>&1
echo "pytest exit $?"
for c in 1 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v45.json 2>> gpurun_out/bench45.err; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_v45.json 2>> gpurun_out/bench45.err
echo done

mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_variants.py -q -x -s -k "variant8" > gpurun_out/pytest_v8_86.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --config 4 --variant 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_v8_86.json 2> gpurun_out/bench_c4_v8_86.err
echo "bench exit $?"
timeout 900 python -m pytest tests/gpu/test_parity.py tests/gpu/test_variants.py -q -x > gpurun_out/pytest_pv86.log 2>&1
echo "pytest2 exit $?"

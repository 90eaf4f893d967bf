mkdir -p gpurun_out
for s in 5 4; do timeout 120 python tools/jitter_check.py $s > gpurun_out/jitter32_s$s.log 2>&1; done
timeout 900 python -m pytest tests/gpu/test_variants.py tests/gpu/test_parity.py -q -x > gpurun_out/pytest32.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v32.json 2> gpurun_out/bench_c5_v32.err
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_v32.json 2>> gpurun_out/bench_c5_v32.err
echo done

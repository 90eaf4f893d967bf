mkdir -p gpurun_out
timeout 1200 python -m pytest tests/gpu/test_parity.py tests/gpu/test_spatial_parity.py -q -x > gpurun_out/pytest38.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_v38.json 2> gpurun_out/bench38.err
echo done

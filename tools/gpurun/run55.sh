mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu55.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_55.json 2> gpurun_out/bench55.err
echo "bench exit $?"

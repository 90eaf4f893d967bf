mkdir -p gpurun_out
timeout 600 python -m pytest tests/gpu/test_recursive_contract.py -q -x -s > gpurun_out/pytest_contract65.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rec65.json 2> gpurun_out/bench_rec65.err
echo "bench exit $?"

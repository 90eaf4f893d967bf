mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1
echo "smoke exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu13.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v13.json 2> gpurun_out/bench_c5_v13.err
for c in 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v13.json 2>> gpurun_out/bench_small_v13.err; done
echo done

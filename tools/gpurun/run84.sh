mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu84.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke84.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench84.json 2> gpurun_out/bench84.err
echo "bench exit $?"
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench84_rec.json 2> gpurun_out/bench84_rec.err
echo "bench rec exit $?"

mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_random_cases.py -q > gpurun_out/pytest_rand39.log 2>&1
echo "random exit $?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu39.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke39.log 2>&1
echo "smoke exit $?"

mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_sweep_parity.py -q -x -s > gpurun_out/pytest_sweep89.log 2>&1
echo "pytest exit $?"

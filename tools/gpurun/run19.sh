# full GPU suite incl. stratified sampler, sweep, recursive, spatial
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -rA > gpurun_out/pytest_gpu19.log 2>&1
echo "pytest exit $?"

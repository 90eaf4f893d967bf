mkdir -p gpurun_out
timeout 600 python -m pytest tests/gpu/test_p2p_two_ranks.py -q -x -s > gpurun_out/pytest_p2p72.log 2>&1
echo "pytest exit $?"

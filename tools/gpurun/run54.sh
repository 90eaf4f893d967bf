mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_parity.py -q -x -k "batch or graph or p2p" > gpurun_out/pytest54.log 2>&1
echo "pytest exit $?"
timeout 600 python tools/batch_bench.py > gpurun_out/batch54.log 2>&1
echo done

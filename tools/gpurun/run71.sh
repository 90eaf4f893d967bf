mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_parity.py -q -x -k "edge_cases" > gpurun_out/pytest_edge71.log 2>&1
echo "pytest exit $?"
timeout 900 python tools/sched_sweep.py --config 5 --groups 0,4,8,37,74 --reps 3 > gpurun_out/sched71.txt 2>&1
echo "sweep exit $?"

mkdir -p gpurun_out
for s in 16; do timeout 300 python tools/profile_run.py --config 5 --samples 28 --reps 4 --engine 1 --sigma $s > gpurun_out/rec43_s$s.log 2>&1; done
timeout 600 python -m pytest tests/gpu/test_recursive_parity.py -q -x > gpurun_out/pytest43.log 2>&1
echo "pytest exit $?"

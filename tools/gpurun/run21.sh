# colour tests + full GPU suite + recursive timing with more reps
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu21.log 2>&1
echo "pytest exit $?"
for s in 2 8 16 32 64; do timeout 300 python tools/profile_run.py --config 5 --samples 28 --reps 4 --engine 1 --sigma $s > gpurun_out/rec21_s$s.log 2>&1; done
echo done

# variants incl. v5 (two samples per pass), full GPU suite, v5 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_variants.py -q -x > gpurun_out/pytest_var22.log 2>&1
echo "variants exit $?"
for v in 2 4; do timeout 300 python tools/profile_run.py --config 5 --samples 64 --reps 3 --variant $v > gpurun_out/var22_$v.log 2>&1; done
for v in 2 4; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_c5_var22_$v.json 2>> gpurun_out/bench22.err; done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu22.log 2>&1
echo "pytest exit $?"

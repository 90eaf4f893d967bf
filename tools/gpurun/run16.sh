# v4b (CW=1, red.add, prefetch) vs CW=2; GPU tests incl. spatial kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu16.log 2>&1
echo "pytest exit $?"
for v in 2 3 1; do timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 64 --reps 3 --variant $v > gpurun_out/var16_$v.log 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v16.json 2> gpurun_out/bench_c5_v16.err
for c in 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v16.json 2>> gpurun_out/bench_small_v16.err; done
echo done

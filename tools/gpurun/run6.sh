mkdir -p gpurun_out
timeout 900 python tools/profile_run.py --config 2 --reps 2 > gpurun_out/v3_sanity.log 2>&1
echo "sanity exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu6.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v4.json 2> gpurun_out/bench_c5_v4.err
for c in 1 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v4.json 2>> gpurun_out/bench_small_v4.err; done
for tr in 1024 2048 4096 8192; do timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 32 --reps 2 --tile-rows $tr > gpurun_out/tile4_$tr.log 2>&1; done
echo done

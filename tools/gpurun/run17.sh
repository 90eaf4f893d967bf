# recursive engine v1 + TMEM consumer (prefetched RMW); GPU tests; sigma sweep
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu17.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v17.json 2> gpurun_out/bench_c5_v17.err
for c in 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v17.json 2>> gpurun_out/bench_small_v17.err; done
for s in 2 4 8 16 32 64; do timeout 300 python tools/profile_run.py --config 5 --samples 16 --reps 2 --engine 1 --sigma $s > gpurun_out/rec17_s$s.log 2>&1; done
for s in 2 4 8 16; do timeout 300 python tools/profile_run.py --config 5 --samples 16 --reps 2 --sigma $s > gpurun_out/fir17_s$s.log 2>&1; done
echo done

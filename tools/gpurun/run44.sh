mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config 5 --samples 28 --reps 4 --engine 1 > gpurun_out/rec44.log 2>&1
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_rec44.json 2> gpurun_out/bench_c5_rec44.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_44.json 2>> gpurun_out/bench_c5_rec44.err
echo done

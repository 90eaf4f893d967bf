# v5 CW=2 default: full GPU suite, bench lines, schedule sweeps, d8 variant 6
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu26.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py > gpurun_out/bench_r01_v5b_full.json 2> gpurun_out/bench_r01_v5b_full.err
echo "bench exit $?"
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v26.json 2>> gpurun_out/bench_small_v26.err; done
timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --variant 6 > gpurun_out/bench_c4_v26_var6.json 2>> gpurun_out/bench_small_v26.err
timeout 600 python tools/sched_sweep.py --config 2 --groups 0,4,8,16,32 --tile-rows 0,256,512 --reps 15 > gpurun_out/sched26_c2.log 2>&1
timeout 600 python tools/sched_sweep.py --config 3 --groups 0,16,32,64 --tile-rows 0,544,1088 --reps 9 > gpurun_out/sched26_c3.log 2>&1
echo done

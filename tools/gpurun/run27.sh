# d8 NA=288, bench pre-warm; GPU suite with new edge cases; bench lines; config-2 ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu27.log 2>&1
echo "pytest exit $?"
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v27.json 2>> gpurun_out/bench_small_v27.err; done
timeout 600 python tools/sched_sweep.py --config 2 --groups 0,4,8,16,32 --tile-rows 0,128,256,512 --reps 15 > gpurun_out/sched27_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 3 -c 1 -o gpurun_out/prof_c2_v27 python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2_v27.log 2>&1
echo "ncu exit $?"

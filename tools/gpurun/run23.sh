# v5 default: full GPU suite + bench lines (configs 5, 2, 3) + launch list + ncu capture of the bench launch
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu23.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py > gpurun_out/bench_r01_v5_full.json 2> gpurun_out/bench_r01_v5_full.err
echo "bench exit $?"
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v23.json 2>> gpurun_out/bench_small_v23.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_v5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_ncu23.log 2>&1
echo "launches exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:mcsf -c 1 -o gpurun_out/prof_c5_v5_bench python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5_v5_bench.log 2>&1
echo "ncu exit $?"

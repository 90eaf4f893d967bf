# v6 default: full suite, bench lines all configs, schedule sweep c3, ncu capture of the bench launch traffic
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu35.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py > gpurun_out/bench_r01_v6_full.json 2> gpurun_out/bench_r01_v6_full.err
echo "bench exit $?"
for c in 1 2 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v35.json 2>> gpurun_out/bench_small_v35.err; done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:mcsf -c 1 --csv --log-file gpurun_out/traffic_v6.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_v6.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_v6.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_ncu35.log 2>&1
echo "ncu exit $?"

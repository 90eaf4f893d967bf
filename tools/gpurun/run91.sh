mkdir -p gpurun_out
timeout 910 python -m pytest tests/gpu/test_variants.py -q -x -s -k "variant8" > gpurun_out/pytest_v8_91.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --config 4 --variant 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_v8_91.json 2> gpurun_out/bench_c4_v8_91.err
echo "bench exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_91_launches.csv python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4_91_ncu.log 2>&1; echo "ll exit $?"

mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu81.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_81.json 2> gpurun_out/bench_c4_81.err
echo "bench c4 exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_81_launches.csv \
  python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4_81_ncu.log 2>&1
echo "launch list exit $?"

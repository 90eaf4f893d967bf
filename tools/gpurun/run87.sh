mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu87.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke87.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench87.json 2> gpurun_out/bench87.err
echo "bench exit $?"
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench87_c4.json 2> gpurun_out/bench87_c4.err
echo "bench c4 exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_87_launches.csv \
  python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4_87_ncu.log 2>&1
echo "launch list exit $?"

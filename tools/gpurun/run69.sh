mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_recursive_parity.py -q -x -s > gpurun_out/pytest_rec69.log 2>&1
echo "pytest exit $?"
for impl in 1; do
  for s in 2 16 64; do
    echo "impl=$impl sigma=$s" >> gpurun_out/rec69.txt
    timeout 300 python tools/profile_run.py --config 5 --engine 1 --rec-impl $impl --sigma $s --samples 28 --reps 5 >> gpurun_out/rec69.txt 2>&1
  done
done
echo "sweep exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rec69_launches.csv \
  python tools/profile_run.py --config 5 --engine 1 --rec-impl 1 --samples 8 --reps 1 > gpurun_out/rec69_ncu1.log 2>&1
echo "launch list exit $?"

# pipelined recursive row kernel: parity + timing + profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_sweep_parity.py -q -x > gpurun_out/pytest_rec20.log 2>&1
echo "pytest exit $?"
for s in 2 16 64; do timeout 300 python tools/profile_run.py --config 5 --samples 16 --reps 2 --engine 1 --sigma $s > gpurun_out/rec20_s$s.log 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rec_ -s 2 -c 2 -o gpurun_out/prof_rec20 python tools/profile_run.py --config 5 --samples 8 --reps 2 --engine 1 > gpurun_out/ncu_rec20.log 2>&1
echo "ncu exit $?"

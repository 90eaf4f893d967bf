# recursive engine profile + sweep tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_sweep_parity.py -q -x > gpurun_out/pytest_sweep18.log 2>&1
echo "pytest exit $?"
timeout 300 python tools/profile_run.py --config 5 --samples 8 --reps 2 --engine 1 > gpurun_out/rec18_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rec_ -s 2 -c 2 -o gpurun_out/prof_rec18 python tools/profile_run.py --config 5 --samples 8 --reps 2 --engine 1 > gpurun_out/ncu_rec18.log 2>&1
echo "ncu exit $?"

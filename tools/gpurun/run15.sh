# v5 consumer rework: GPU parity tests, benches, ncu full capture
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu15.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v5.json 2> gpurun_out/bench_c5_v5.err
echo "bench exit $?"
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v5.json 2>> gpurun_out/bench_small_v5.err; done
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/prof_plain15.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 -o gpurun_out/prof_c5_v5 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/ncu_c5_v5.log 2>&1
echo "ncu exit $?"

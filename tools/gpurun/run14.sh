# r01 v4 validation: smoke, GPU parity tests, full bench line, launch list, full ncu capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1
echo "smoke exit $?"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu14.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py > gpurun_out/bench_r01_v4_full.json 2> gpurun_out/bench_r01_v4_full.err
echo "bench exit $?"
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v4.json 2>> gpurun_out/bench_small_v4.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_v4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_ncu14.log 2>&1
echo "launches exit $?"
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/prof_plain14.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 -o gpurun_out/prof_c5_v4 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/ncu_c5_v4.log 2>&1
echo "ncu exit $?"

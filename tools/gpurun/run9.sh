mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 900 python bench.py > gpurun_out/bench_r01_full.json 2> gpurun_out/bench_r01_full.err
echo "bench exit $?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_ncu.log 2>&1
echo "launches exit $?"
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 --tile-rows 8192 --groups 4 > gpurun_out/prof_plain9.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf_fused -s 1 -c 1 -o gpurun_out/prof_c5_v3b python tools/profile_run.py --config 5 --rows 8192 --samples 16 --tile-rows 8192 --groups 4 > gpurun_out/ncu_c5_v3b.log 2>&1
echo "ncu exit $?"

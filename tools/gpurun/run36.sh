mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/prof_plain36.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 -o gpurun_out/prof_c5_v6 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/ncu_c5_v6.log 2>&1
echo "ncu exit $?"
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_recursive.json 2> gpurun_out/bench_c5_recursive.err
timeout 600 python tools/paper_experiments.py --which lab --reps 10 --out gpurun_out/lab36.json > gpurun_out/lab36.log 2>&1
echo done

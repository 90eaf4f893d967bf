mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu33.log 2>&1
echo "pytest exit $?"
timeout 900 python tools/paper_experiments.py --which table1 --reps 15 --out gpurun_out/table1_r33.json > gpurun_out/table1_r33.log 2>&1
for c in 1 2 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v33.json 2>> gpurun_out/bench_small_v33.err; done
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/prof_plain33.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 -o gpurun_out/prof_c5_v5c python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/ncu_c5_v5c.log 2>&1
echo "ncu exit $?"

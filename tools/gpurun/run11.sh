mkdir -p gpurun_out
timeout 900 python tools/profile_run.py --config 5 --rows 8192 --samples 32 --reps 2 > gpurun_out/v6_c5.log 2>&1
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v6.json 2>> gpurun_out/bench_small_v6.err; done
timeout 900 python tools/accuracy_report.py > gpurun_out/accuracy.jsonl 2> gpurun_out/accuracy.err
echo "acc exit $?"

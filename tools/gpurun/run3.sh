set -x
mkdir -p gpurun_out
timeout 600 python tools/profile_run.py --config 5 --rows 1024 --samples 64 > gpurun_out/prof_plain3.log 2>&1
echo "prof exit $?"
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5_v2.json 2> gpurun_out/bench_c5_v2.err
echo "bench exit $?"
for c in 1 2 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c${c}_v2.json 2>> gpurun_out/bench_small_v2.err; done
echo done

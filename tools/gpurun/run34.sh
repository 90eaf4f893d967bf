# v6 (dedicated modulation warps): parity + timing vs v5c
mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_variants.py -q -x > gpurun_out/pytest_var34.log 2>&1
echo "variants exit $?"
for v in 4 6; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_c5_var34_$v.json 2>> gpurun_out/bench34.err; done
echo done

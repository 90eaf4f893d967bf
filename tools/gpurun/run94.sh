mkdir -p gpurun_out
for v in 0 6 0 6; do
  timeout 300 python bench.py --config 2 --variant $v --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/b94_c2.jsonl 2>> gpurun_out/b94.err
  echo "v$v exit $?"
done
timeout 600 python -m pytest tests/gpu/test_variants.py -q -x -k "config2" > gpurun_out/pytest_v94.log 2>&1
echo "pytest exit $?"

mkdir -p gpurun_out
for s in 2 5 8; do for v in 1 8; do
  timeout 300 python bench.py --config 4 --sigma $s --variant $v --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b80_s${s}_v${v}.json 2>> gpurun_out/b80.err
  echo "s$s v$v exit $?"
done; done
timeout 900 python -m pytest tests/gpu/test_variants.py -q -x -k "variant8" > gpurun_out/pytest_v8_80.log 2>&1
echo "pytest exit $?"

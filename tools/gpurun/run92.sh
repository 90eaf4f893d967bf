mkdir -p gpurun_out
for c in 2 3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b92_c$c.json 2>> gpurun_out/b92.err
  echo "c$c exit $?"
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b92_c5.json 2>> gpurun_out/b92.err
echo "c5 exit $?"
timeout 900 python -m pytest tests/gpu/test_parity.py tests/gpu/test_variants.py -q -x > gpurun_out/pytest_pv92.log 2>&1
echo "pytest exit $?"

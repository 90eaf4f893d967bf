mkdir -p gpurun_out
for c in 1 2; do
  for v in 0 2; do
    timeout 300 python bench.py --config $c --variant $v --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b56_c${c}_v${v}.json 2>> gpurun_out/b56.err
    echo "c$c v$v exit $?"
  done
done
timeout 300 python tools/batch_bench.py > gpurun_out/batch56.log 2>&1; echo "batch exit $?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu56.log 2>&1
echo "pytest exit $?"

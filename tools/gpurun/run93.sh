mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu93.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke93.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench93.json 2> gpurun_out/bench93.err
echo "bench exit $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench93_ref.json 2> gpurun_out/bench93_ref.err
echo "ref exit $?"
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench93_c$c.json 2>> gpurun_out/bench93_cx.err
  echo "c$c exit $?"
done
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench93_rec.json 2> gpurun_out/bench93_rec.err
echo "rec exit $?"

mkdir -p gpurun_out
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rec62.json 2> gpurun_out/bench_rec62.err
echo "bench exit $?"
timeout 900 python tools/paper_experiments.py --which table1 --out gpurun_out/table1_r62.json > gpurun_out/table1_r62.log 2>&1
echo "table1 exit $?"

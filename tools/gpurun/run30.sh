mkdir -p gpurun_out
timeout 900 python tools/paper_experiments.py --which table1 --reps 15 --out gpurun_out/table1_r30.json > gpurun_out/table1_r30.log 2>&1
echo "exit $?"

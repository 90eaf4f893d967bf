mkdir -p gpurun_out
timeout 900 python tools/paper_experiments.py --which table1 --out gpurun_out/table1_r70.json > gpurun_out/table1_r70.log 2>&1
echo "table1 exit $?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu70.log 2>&1
echo "pytest exit $?"

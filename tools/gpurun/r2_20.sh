# round 2, call 20: the paper's experiments (Table 1, Fig. 5) and the accuracy report re-run with the
# round-2 kernels (new exact filter, persistent schedule)
mkdir -p gpurun_out
timeout 1200 python tools/paper_experiments.py --which table1 --out gpurun_out/r2_20_table1.json > gpurun_out/r2_20_table1.log 2>&1
echo "table1 exit $?"; tail -8 gpurun_out/r2_20_table1.log
timeout 1500 python tools/accuracy_report.py > gpurun_out/r2_20_accuracy.jsonl 2> gpurun_out/r2_20_accuracy.err
echo "accuracy exit $?"; cat gpurun_out/r2_20_accuracy.jsonl | cut -c1-300

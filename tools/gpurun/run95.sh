mkdir -p gpurun_out
timeout 1200 python tools/accuracy_report.py > gpurun_out/accuracy95.jsonl 2> gpurun_out/accuracy95.err
echo "acc exit $?"

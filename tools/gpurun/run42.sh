mkdir -p gpurun_out
timeout 900 python tools/accuracy_report.py > gpurun_out/accuracy42.jsonl 2> gpurun_out/accuracy42.err
echo "acc exit $?"

mkdir -p gpurun_out
timeout 900 python tools/scaling_projection.py > gpurun_out/scaling51.log 2>&1
echo "exit $?"

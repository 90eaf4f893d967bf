# round 2, call 21: per-rank work of the N-GPU partitions timed on one GPU (persistent schedule)
mkdir -p gpurun_out
timeout 1500 python tools/scaling_projection.py > gpurun_out/r2_21_scaling.txt 2>&1
echo "exit $?"; cat gpurun_out/r2_21_scaling.txt

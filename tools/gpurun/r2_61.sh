# round 2, call 61: ncu --set full of rect_tc2_kernel (tensor-core pass 2)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_tc2 -c 1 \
    -o gpurun_out/r2_61_tc2 -f python tools/profile_run.py --config 5 --engine 1 --rec-tc 1 --samples 16 --reps 1 > gpurun_out/r2_61_ncu.log 2>&1
echo "ncu exit $?"

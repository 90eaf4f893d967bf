# round 2, call 46: ncu --set full of rect_vscan_kernel (rec_impl 3)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_vscan -c 1 \
    -o gpurun_out/r2_46_vscan -f python tools/profile_run.py --config 5 --engine 1 --rec-impl 3 --samples 16 --reps 1 > gpurun_out/r2_46_ncu.log 2>&1
echo "ncu exit $?"

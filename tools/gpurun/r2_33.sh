# round 2, call 33: ncu --set full of the v6 kernel on config 3 (R = 30, classic grid) and config 4 (variant 8)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 \
  -o gpurun_out/r2_33_v6_c3 -f python tools/profile_run.py --config 3 --reps 2 > gpurun_out/r2_33_ncu_c3.log 2>&1
echo "ncu c3 exit $?"

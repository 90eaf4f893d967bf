# round 2, call 12: ncu of the v6 kernel on config 2 (persistent + OV) and config 5 (persistent)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 \
  -o gpurun_out/r2_12_v6_c2 -f python tools/profile_run.py --config 2 --reps 2 > gpurun_out/r2_12_ncu_c2.log 2>&1
echo "ncu c2 exit $?"; tail -2 gpurun_out/r2_12_ncu_c2.log

mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mcsf_tmem8 -c 2 -o gpurun_out/c4v8_88_full \
  python tools/profile_run.py --config 4 --reps 1 > gpurun_out/c4v8_88_ncu.log 2>&1
echo "ncu exit $?"

mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rec58_launches.csv \
  python tools/profile_run.py --config 5 --engine 1 --rec-impl 1 --samples 8 --reps 1 > gpurun_out/rec58_ncu1.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rect_ -c 4 -o gpurun_out/rec58_full \
  python tools/profile_run.py --config 5 --engine 1 --rec-impl 1 --samples 8 --reps 1 > gpurun_out/rec58_ncu2.log 2>&1
echo "full exit $?"

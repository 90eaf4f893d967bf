mkdir -p gpurun_out
timeout 600 python tools/sched_sweep.py --config 4 --variant 8 --groups 0,16,32,37,64 --tile-rows 0,512 --reps 5 > gpurun_out/sched76.txt 2>&1
echo "sweep exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4v8_76_launches.csv \
  python tools/profile_run.py --config 4 --variant 8 --reps 1 > gpurun_out/c4v8_76_ncu1.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mcsf_tmem8 -c 3 -o gpurun_out/c4v8_76_full \
  python tools/profile_run.py --config 4 --variant 8 --reps 1 > gpurun_out/c4v8_76_ncu2.log 2>&1
echo "ncu full exit $?"

mkdir -p gpurun_out
timeout 900 python tools/sched_sweep.py --config 4 --groups 0,32,37,40,48,64,74,111,148 --tile-rows 0,512 --reps 5 > gpurun_out/sched74.txt 2>&1
echo "sweep exit $?"

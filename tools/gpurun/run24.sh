mkdir -p gpurun_out
timeout 600 python tools/sched_sweep.py --config 5 --groups 0,4,8,16,19,32,37 --reps 3 > gpurun_out/sched24_c5.log 2>&1
timeout 300 python tools/sched_sweep.py --config 3 --groups 0,8,16,32,64 --tile-rows 0,540,1088 --reps 5 > gpurun_out/sched24_c3.log 2>&1
timeout 300 python tools/sched_sweep.py --config 2 --groups 0,4,8,16,32,64 --tile-rows 0,128,256,512 --reps 5 > gpurun_out/sched24_c2.log 2>&1
echo done

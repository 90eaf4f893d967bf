mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_variants.py -q -x > gpurun_out/pytest_var25.log 2>&1
echo "variants exit $?"
timeout 900 python tools/sched_sweep.py --config 5 --groups 4,16,32,64,128 --reps 3 --variant 4 > gpurun_out/sched25_v4.log 2>&1
timeout 900 python tools/sched_sweep.py --config 5 --groups 4,16,32,64,128 --reps 3 --variant 5 > gpurun_out/sched25_v5.log 2>&1
timeout 600 python tools/sched_sweep.py --config 3 --groups 16,32,64 --reps 5 --variant 5 > gpurun_out/sched25_c3v5.log 2>&1
timeout 600 python tools/sched_sweep.py --config 3 --groups 16,32,64 --reps 5 --variant 4 > gpurun_out/sched25_c3v4.log 2>&1
echo done

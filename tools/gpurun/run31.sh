mkdir -p gpurun_out
for s in 5 4; do timeout 120 python tools/jitter_check.py $s > gpurun_out/jitter_s$s.log 2>&1; done
nvidia-smi -q -d PERFORMANCE,CLOCK,POWER > gpurun_out/smi_q.txt 2>&1
echo done

# round 2, call 50: tcgen05 tf32 probe (A from TMEM, B K-major no-swizzle in shared memory)
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/r2_50_probe.log 2>&1; echo "probe exit $?"; cat gpurun_out/r2_50_probe.log | tail -12

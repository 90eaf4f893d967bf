mkdir -p gpurun_out
timeout 300 python tools/sig4_check.py > gpurun_out/sig4.log 2>&1
timeout 300 python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/prof_plain29.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 1 -c 1 -o gpurun_out/prof_c5_v5b python tools/profile_run.py --config 5 --rows 8192 --samples 16 > gpurun_out/ncu_c5_v5b.log 2>&1
echo "ncu exit $?"

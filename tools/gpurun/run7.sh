mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config 5 --rows 1024 --samples 64 --tile-rows 1024 --groups 1 > gpurun_out/prof_plain7.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mcsf_fused -s 1 -c 1 -o gpurun_out/prof_c5_v3 python tools/profile_run.py --config 5 --rows 1024 --samples 64 --tile-rows 1024 --groups 1 > gpurun_out/ncu_c5_v3.log 2>&1
echo "ncu exit $?"

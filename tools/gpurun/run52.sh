mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 3 -c 1 -o gpurun_out/prof_c3_v6 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
echo "ncu exit $?"

mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke37.log 2>&1
echo "smoke exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mcsf -s 3 -c 1 -o gpurun_out/prof_c4_v6 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1
echo "ncu exit $?"

# round 2, call 24: ncu --set full of the bench's fused launch (config 5, persistent schedule), examples
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:mcsf -c 1 \
  -o gpurun_out/r2_24_v6_c5 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/r2_24_ncu.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/r2_24_ncu.log
timeout 300 python examples/filter_torch.py > gpurun_out/r2_24_example_py.log 2>&1; echo "example py exit $?"; tail -3 gpurun_out/r2_24_example_py.log

# round 2, call 3: the tiled exact (direct) filter: parity vs O3, timing vs roofline, ncu
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/gpu/test_direct_parity.py tests/gpu/test_parity.py tests/gpu/test_spatial_parity.py -k direct -q -x > gpurun_out/r2_03_pytest.log 2>&1
echo "pytest exit $?"; tail -5 gpurun_out/r2_03_pytest.log
timeout 600 python tools/direct_bench.py --json gpurun_out/r2_03_direct_bench.json > gpurun_out/r2_03_direct_bench.log 2>&1
echo "bench exit $?"; cat gpurun_out/r2_03_direct_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:direct_tiled --launch-skip 3 --launch-count 1 \
  -o gpurun_out/r2_03_direct_c2 -f python tools/direct_bench.py --only cfg2 --reps 1 > gpurun_out/r2_03_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/r2_03_ncu.log

# round 2, call 4: packed-pair (FFMA2) exact filter, CTA height sweep, parity, ncu
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/gpu/test_direct_parity.py tests/gpu/test_parity.py tests/gpu/test_spatial_parity.py -k direct -q -x > gpurun_out/r2_04_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r2_04_pytest.log
for rows in 0 4 8 16; do
timeout 600 python tools/direct_bench.py --rows $rows --json gpurun_out/r2_04_direct_rows$rows.json > gpurun_out/r2_04_direct_rows$rows.log 2>&1
echo "bench rows=$rows exit $?"; python -c "
import json; [print(r['case'], r['direct_rows'], round(r['ms'],4), round(r['frac_of_roofline'],3)) for r in json.load(open('gpurun_out/r2_04_direct_rows$rows.json'))]"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:direct_tiled --launch-skip 3 --launch-count 1 \
  -o gpurun_out/r2_04_direct_c2 -f python tools/direct_bench.py --only cfg2 --reps 1 > gpurun_out/r2_04_ncu.log 2>&1
echo "ncu exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:direct_tiled --launch-skip 3 --launch-count 1 \
  -o gpurun_out/r2_04_direct_c3 -f python tools/direct_bench.py --only cfg3 --reps 1 > gpurun_out/r2_04_ncu3.log 2>&1
echo "ncu3 exit $?"

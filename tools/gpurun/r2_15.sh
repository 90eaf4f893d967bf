# round 2, call 15: persistent shares cut on whole passes when they span >= 50 passes (L2 reuse of f)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_variants.py -q -x -k "persistent" > gpurun_out/r2_15_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r2_15_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_15_bench_c5.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2_15_bench_c5.json').read().strip().splitlines()[-1]); print('cfg5', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'groups', d['config']['groups'], 'persistent', d['config']['persistent'])"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:mcsf -c 1 --csv --log-file gpurun_out/r2_15_traffic_c5.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/r2_15_traffic.log 2>&1
echo "traffic exit $?"; grep -E "dram__bytes|duration" gpurun_out/r2_15_traffic_c5.csv | awk -F'","' '{print $13, $15}'

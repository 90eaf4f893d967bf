# round 2, call 78: persistent tensor-core column scan (virtual blocks)
# memory set up once) -- recursive parity incl. other d, bench, launch list
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/gpu/test_recursive_parity.py -q -x > gpurun_out/r2_78_pytest.log 2>&1
echo "tests exit $?"; tail -1 gpurun_out/r2_78_pytest.log
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_78_rec.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2_78_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_78_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_78_launches.csv 2>/dev/null | sed -n 3,6p

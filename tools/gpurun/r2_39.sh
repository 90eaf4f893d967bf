# round 2, call 39: rec_impl 3 (virtual-line row blur folded into the column scan) -- recursive parity on
# all four implementations, bench rec_impl 2 vs 3, launch list
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_recursive_contract.py -q -x > gpurun_out/r2_39_pytest.log 2>&1
echo "recursive tests exit $?"; tail -15 gpurun_out/r2_39_pytest.log
for ri in 2 3; do
  timeout 600 python bench.py --engine 1 --rec-impl $ri --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_39_rec_$ri.json 2>gpurun_out/r2_39_rec_$ri.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_39_rec_$ri.json').read().strip().splitlines()[-1]); print('rec_impl $ri', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_39_launches_3.csv \
    python tools/profile_run.py --config 5 --engine 1 --rec-impl 3 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_39_launches_3.csv 2>/dev/null | head -12

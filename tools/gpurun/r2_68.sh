# round 2, call 68: tensor-core pass 0 summaries (option rec_tc0) -- parity, A/B bench, launch list
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py -q -x -k "vlines_tc_all" > gpurun_out/r2_68_pytest.log 2>&1
echo "tests exit $?"; tail -3 gpurun_out/r2_68_pytest.log
for v in 0 1; do
  timeout 600 python bench.py --engine 1 --rec-tc0 $v --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_68_rec_$v.json 2>gpurun_out/r2_68_rec_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_68_rec_$v.json').read().strip().splitlines()[-1]); print('tc0 $v', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])" || tail -3 gpurun_out/r2_68_rec_$v.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_68_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --rec-tc0 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_68_launches.csv 2>/dev/null | sed -n 3,7p

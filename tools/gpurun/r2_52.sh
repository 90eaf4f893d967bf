# round 2, call 52: tensor-core pass 2 with the two M halves as independent pipelines -- recursive parity on every implementation incl.
# vlines_tc, contract tests, bench rec_tc 0 vs 1, launch list
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_recursive_contract.py -q > gpurun_out/r2_52_pytest.log 2>&1
echo "recursive tests exit $?"; grep -E "passed|failed|Error|assert" gpurun_out/r2_52_pytest.log | head -20
for tc in 0 1; do
  timeout 600 python bench.py --engine 1 --rec-tc $tc --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_52_rec_tc$tc.json 2>gpurun_out/r2_52_rec_tc$tc.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_52_rec_tc$tc.json').read().strip().splitlines()[-1]); print('rec_tc $tc', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])" || tail -3 gpurun_out/r2_52_rec_tc$tc.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_52_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --rec-tc 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_52_launches.csv 2>/dev/null | head -10

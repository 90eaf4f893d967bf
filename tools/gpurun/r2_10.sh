# round 2, call 10: persistent schedule of the v6 kernel: parity, then config 1/2/3/5 timing (auto vs classic)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_variants.py -q -x -k "persistent" > gpurun_out/r2_10_pytest.log 2>&1
echo "pytest exit $?"; tail -4 gpurun_out/r2_10_pytest.log
for cfg in 2 1 3 5; do
  steps=20; [ $cfg = 5 ] && steps=5
  for pm in 0 1; do
    timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e --persistent $pm > gpurun_out/r2_10_c${cfg}_p$pm.json 2> gpurun_out/r2_10_c${cfg}_p$pm.err
    python -c "
import json; d=json.loads(open('gpurun_out/r2_10_c${cfg}_p$pm.json').read().strip().splitlines()[-1]); print('cfg$cfg persistent=$pm', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'kernel_ms %.4f'%d['roofline']['fused_ms_per_launch'], 'groups', d['config']['groups'], 'used', d['config']['persistent'])"
  done
done

# round 2, call 11: pass overlap (OV: R <= 24) + persistent schedule: parity of every v6 radius, timing
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/gpu/test_variants.py tests/gpu/test_parity.py -q -x > gpurun_out/r2_11_pytest.log 2>&1
echo "pytest exit $?"; tail -4 gpurun_out/r2_11_pytest.log
for cfg in 2 1 3; do
  for pm in 0 1; do
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --persistent $pm > gpurun_out/r2_11_c${cfg}_p$pm.json 2> gpurun_out/r2_11_c${cfg}_p$pm.err
    python -c "
import json; d=json.loads(open('gpurun_out/r2_11_c${cfg}_p$pm.json').read().strip().splitlines()[-1]); print('cfg$cfg persistent=$pm', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'kernel_ms %.4f'%d['roofline']['fused_ms_per_launch'], 'groups', d['config']['groups'], 'used', d['config']['persistent'])"
  done
done
for pm in 0 2; do
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --persistent $pm > gpurun_out/r2_11_c5_p$pm.json 2> gpurun_out/r2_11_c5_p$pm.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_11_c5_p$pm.json').read().strip().splitlines()[-1]); print('cfg5 persistent=$pm', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'kernel_ms %.4f'%d['roofline']['fused_ms_per_launch'], 'groups', d['config']['groups'], 'used', d['config']['persistent'])"
done

# round 2, call 80: recursive engine, batch k+1's pass 0 beside batch k's scans (option rec_overlap):
# bitwise-vs-one-stream tests, then the config-5 A/B (0 / 1 high-priority aux stream / 2 default priority)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/gpu/test_recursive_parity.py -q -x -k "overlap or config_full" > gpurun_out/r2_80_pytest.log 2>&1
echo "tests exit $?"; tail -2 gpurun_out/r2_80_pytest.log
for ov in 0 1 2 0 1 2; do
  timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --rec-overlap $ov > gpurun_out/r2_80_rec_ov$ov.json 2>gpurun_out/r2_80_rec_ov$ov.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_80_rec_ov$ov.json').read().strip().splitlines()[-1]); print('ov $ov', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done

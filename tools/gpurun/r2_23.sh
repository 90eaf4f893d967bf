# round 2, call 23: split fill overlap (HROWS = min(2A, TMEM cap); the first HROWS - A fill rows of a
# pass written while the previous pass's last chunk is read): parity (default + checked build), timing
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/gpu/test_variants.py tests/gpu/test_parity.py -q -x > gpurun_out/r2_23_pytest.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/r2_23_pytest.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 1500 python -m pytest tests/gpu/test_variants.py tests/gpu/test_parity.py -q -x > gpurun_out/r2_23_pytest_checked.log 2>&1
echo "checked exit $?"; tail -2 gpurun_out/r2_23_pytest_checked.log
for cfg in 3 2 5; do
  steps=20; [ $cfg = 5 ] && steps=5
  timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_23_c$cfg.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_23_c$cfg.json').read().strip().splitlines()[-1]); print('cfg$cfg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'groups', d['config']['groups'], 'persistent', d['config']['persistent'])"
done

# round 2, call 72: tensor-core recursion for d != 3 -- recursive parity (all fixtures) + other-d tests,
# config-5 recursive bench (d = 3 unchanged?)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_recursive_contract.py -q -s -k "other_channel or vlines_tc" > gpurun_out/r2_72_pytest.log 2>&1
echo "tests exit $?"; grep -E "passed|failed|^d [0-9]|Error" gpurun_out/r2_72_pytest.log | head -20
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_72_rec.json 2>gpurun_out/r2_72_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_72_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
for c in 4; do
  timeout 600 python bench.py --config 4 --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_72_rec_c4.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_72_rec_c4.json').read().strip().splitlines()[-1]); print('rec c4 (d=8)', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
done

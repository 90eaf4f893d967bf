# round 2, call 84: tensor-core pass 2 transpose rows at pitch 36 with float4 stores (libbfvec_trp36.so)
# vs pitch 33 scalar stores (libbfvec_tr33.so, -DBFVEC_TC_TR33): recursive parity on the trp36 build, config-5 A/B
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_trp36.so timeout 900 python -m pytest tests/gpu/test_recursive_parity.py -q -x -k "vlines_tc" > gpurun_out/r2_84_pytest.log 2>&1
echo "tests exit $?"; tail -n 1 gpurun_out/r2_84_pytest.log
for v in trp36 tr33 trp36 tr33; do
  BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$v.so timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_84_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_84_$v.json').read().strip().splitlines()[-1]); print('$v', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done
for v in trp36 tr33; do
  BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rect_tc2 --csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 2>/dev/null | grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' | sed "s/^/$v /"
done

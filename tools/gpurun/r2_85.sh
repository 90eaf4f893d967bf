# round 2, call 85: pass 2 f tile and (cos, sin) planes at pitch 36 with float4 row-operand reads
# (libbfvec_rowv4.so, -DBFVEC_TC_ROWV4) vs the pitch-36 transposes alone (libbfvec_trp36.so)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_rowv4.so timeout 900 python -m pytest tests/gpu/test_recursive_parity.py -q -x -k "vlines_tc" > gpurun_out/r2_85_pytest.log 2>&1
echo "tests exit $?"; tail -n 1 gpurun_out/r2_85_pytest.log
for v in rowv4 trp36 rowv4 trp36; do
  BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$v.so timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_85_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_85_$v.json').read().strip().splitlines()[-1]); print('$v', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done
for v in rowv4 trp36; do
  BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rect_tc2 --csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 2>/dev/null | grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' | sed "s/^/$v /"
done

# round 2, call 32: recursive pass 2 compiled for 3 CTAs per SM (A/B vs 4)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_recursive_contract.py tests/gpu/test_sweep_parity.py tests/gpu/test_color_parity.py -q -x > gpurun_out/r2_32_pytest.log 2>&1
echo "recursive tests exit $?"; tail -2 gpurun_out/r2_32_pytest.log
for lib in main p2m3; do
  if [ $lib = p2m3 ]; then export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_p2m3.so; else unset BFVEC_LIB; fi
  timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_32_rec_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_32_rec_$lib.json').read().strip().splitlines()[-1]); print('$lib', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_32_launches_$lib.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
done

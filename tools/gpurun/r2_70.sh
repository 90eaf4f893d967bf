# round 2, call 70: tensor-core pass 2, accumulate: cos / sin column loaded while the tensor-memory load is in flight
# waits polled without a suspend hint (A/B vs BFVEC_TC_SLEEP); recursive parity, bench, launch lists
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py -q -k "vlines_tc" > gpurun_out/r2_70_pytest.log 2>&1
echo "tc parity exit $?"; grep -E "passed|failed" gpurun_out/r2_70_pytest.log
for lib in main; do
  if [ $lib = main ]; then unset BFVEC_LIB; else export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$lib.so; fi
  timeout 600 python bench.py --engine 1 --rec-tc 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_70_rec_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_70_rec_$lib.json').read().strip().splitlines()[-1]); print('$lib', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_70_launches_$lib.csv \
    python tools/profile_run.py --config 5 --engine 1 --rec-tc 1 --samples 16 --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r2_70_launches_$lib.csv 2>/dev/null | sed -n 3,3p
done

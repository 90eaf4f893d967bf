# round 2, call 28: stability -- the whole GPU suite three times on the default build and once on
# the checked build (flakes would show up as a failure in one repetition), two bench repetitions
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
for i in 1 2 3; do
  timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r2_28_suite_$i.log 2>&1
  echo "suite $i exit $?"; tail -1 gpurun_out/r2_28_suite_$i.log
done
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2_28_suite_checked.log 2>&1
echo "checked suite exit $?"; tail -1 gpurun_out/r2_28_suite_checked.log; grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_28_suite_checked.log
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_28_bench_$i.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_28_bench_$i.json').read().strip().splitlines()[-1]); print('bench $i', '%.5g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], d['clocks'])"
done

# round 2, call 13: full GPU suite on the default build and on the checked build (sanitizer stand-in),
# smoke(), then the default bench (config 5, all legs) and configs 1-4
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_13_suite_default.log 2>&1
echo "default suite exit $?"; tail -3 gpurun_out/r2_13_suite_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2_13_suite_checked.log 2>&1
echo "checked suite exit $?"; tail -3 gpurun_out/r2_13_suite_checked.log
grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_13_suite_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_13_smoke.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_13_bench_c5.json 2> gpurun_out/r2_13_bench_c5.err
echo "bench c5 exit $?"; tail -c 600 gpurun_out/r2_13_bench_c5.json
for cfg in 1 2 3 4; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 > gpurun_out/r2_13_bench_c$cfg.json 2> gpurun_out/r2_13_bench_c$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_13_bench_c$cfg.json').read().strip().splitlines()[-1]); print('cfg$cfg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], 'persistent', d['config']['persistent'])"
done

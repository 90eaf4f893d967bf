# round 2, call 30: final state (after the recursive-engine changes) -- whole GPU suite (default and checked builds), smoke, bench configs
# 1-5 with every leg, the reference arm, the C examples
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_30_suite_default.log 2>&1
echo "default suite exit $?"; tail -2 gpurun_out/r2_30_suite_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2_30_suite_checked.log 2>&1
echo "checked suite exit $?"; tail -2 gpurun_out/r2_30_suite_checked.log; grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_30_suite_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_30_smoke.log 2>&1; echo "smoke exit $?"
for ex in filter_host filter_frames; do
  gcc -O2 -I include examples/$ex.c -L paper_1605_02164_b200 -lbfvec -Wl,-rpath,$PWD/paper_1605_02164_b200 -lm -o /tmp/$ex && /tmp/$ex > gpurun_out/r2_30_$ex.log 2>&1; echo "$ex exit $?"; cat gpurun_out/r2_30_$ex.log
done
timeout 900 python bench.py > gpurun_out/r2_30_bench_c5.json 2> gpurun_out/r2_30_bench_c5.err; echo "bench c5 exit $?"
for cfg in 1 2 3 4; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 > gpurun_out/r2_30_bench_c$cfg.json 2> gpurun_out/r2_30_bench_c$cfg.err; echo "bench c$cfg exit $?"
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_30_reference.json 2> gpurun_out/r2_30_reference.err; echo "reference exit $?"
for c in 1 2 3 4 5; do python -c "
import json; d=json.loads(open('gpurun_out/r2_30_bench_c$c.json').read().strip().splitlines()[-1]); print('cfg$c', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], d['clocks'])"; done
tail -c 700 gpurun_out/r2_30_reference.json

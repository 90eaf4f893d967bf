# round 2, call 86: final tree (pass 2 at pitch 36: float4 transposes and row-operand reads) -- whole GPU suite default + checked, smoke, FIR bench config 5, recursive bench with e2e
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_86_suite_default.log 2>&1
echo "default suite exit $?"; tail -1 gpurun_out/r2_86_suite_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_86_suite_checked.log 2>&1
echo "checked suite exit $?"; tail -1 gpurun_out/r2_86_suite_checked.log; grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_86_suite_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_86_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r2_86_bench_c5.json 2> gpurun_out/r2_86_bench_c5.err; echo "bench c5 exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_86_bench_c5.json').read().strip().splitlines()[-1]); print('cfg5', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_86_rec.json 2>gpurun_out/r2_86_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_86_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'])"

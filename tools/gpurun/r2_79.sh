# round 2, call 79: final tree (persistent tensor-core pass 2) -- whole GPU suite default + checked, smoke, benches, reference arm, Table 1
# bench config 5, recursive bench, reference arm, Table 1 with the tensor-core recursive engine
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_79_suite_default.log 2>&1
echo "default suite exit $?"; tail -1 gpurun_out/r2_79_suite_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_79_suite_checked.log 2>&1
echo "checked suite exit $?"; tail -1 gpurun_out/r2_79_suite_checked.log; grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_79_suite_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_79_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r2_79_bench_c5.json 2> gpurun_out/r2_79_bench_c5.err; echo "bench c5 exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_79_bench_c5.json').read().strip().splitlines()[-1]); print('cfg5', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_79_rec.json 2>gpurun_out/r2_79_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_79_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'])"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_79_reference.json 2> gpurun_out/r2_79_reference.err; echo "reference exit $?"
timeout 600 python tools/paper_experiments.py --which table1 --out gpurun_out/r2_79_table1.json > gpurun_out/r2_79_table1.log 2>&1; echo "table1 exit $?"

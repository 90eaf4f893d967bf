# round 2, call 59: tensor-core pass 2 the default for d = 3 -- whole GPU suite, smoke, recursive bench
# (rec_tc 1 / 0, e2e), sigma sweep, launch list
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_59_suite.log 2>&1
echo "suite exit $?"; tail -2 gpurun_out/r2_59_suite.log; grep -E "^FAILED|Error" gpurun_out/r2_59_suite.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_59_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r2_59_smoke.log
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_59_rec.json 2>gpurun_out/r2_59_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_59_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], d['roofline']['kernel'], 'e2e %.4g'%d['e2e']['value'])"
for sg in 2 64; do
  timeout 600 python bench.py --engine 1 --sigma $sg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_59_rec_s$sg.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_59_rec_s$sg.json').read().strip().splitlines()[-1]); print('sigma $sg', '%.4g'%d['value'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_59_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_59_launches.csv 2>/dev/null | head -8

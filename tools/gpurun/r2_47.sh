# round 2, call 47: rec_impl 2 = virtual-line blur inside the column scan (vline kernel removed), pass 2
# at 3 CTAs/SM with entering states converted at their use -- whole GPU suite, smoke, recursive bench
# (e2e too), launch list, ncu --set full of pass 2
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_47_suite.log 2>&1
echo "suite exit $?"; tail -2 gpurun_out/r2_47_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_47_smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/r2_47_smoke.log
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_47_rec.json 2>gpurun_out/r2_47_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_47_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], d['roofline']['kernel'], 'e2e %.4g'%d['e2e']['value'])"
for sg in 2 16 64; do
  timeout 600 python bench.py --engine 1 --sigma $sg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_47_rec_s$sg.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_47_rec_s$sg.json').read().strip().splitlines()[-1]); print('sigma $sg', '%.4g'%d['value'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_47_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_47_launches.csv 2>/dev/null | head -10
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_tile_kernel -s 1 -c 1 \
    -o gpurun_out/r2_47_p2 -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_47_ncu_p2.log 2>&1
echo "ncu p2 exit $?"

# round 2, call 81: recursive engine batch-size A/B (16 auto / 32 / 48), launch list and ncu --set full of
# the persistent tensor-core pass 2 and of pass 0 (current tree)
mkdir -p gpurun_out
for nb in 0 32 48 0 32 48; do
  timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --rec-batch $nb > gpurun_out/r2_81_rec_nb$nb.json 2>gpurun_out/r2_81_rec_nb$nb.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_81_rec_nb$nb.json').read().strip().splitlines()[-1]); print('nb $nb', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_81_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_81_launches.csv 2>/dev/null | head -12
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_tc2 -c 1 \
    -o gpurun_out/r2_81_tc2 -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_81_ncu_tc2.log 2>&1
echo "ncu tc2 exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_tile -c 1 \
    -o gpurun_out/r2_81_p0 -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_81_ncu_p0.log 2>&1
echo "ncu p0 exit $?"

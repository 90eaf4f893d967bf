# round 2, call 82: recursive engine batch cap 48 (auto = min(48, 40 % of free memory)): bench auto vs
# forced 16 / 64, sigma 2 and 64 with auto, first-call cost (fresh plan, 3 reps) auto vs 16
mkdir -p gpurun_out
for nb in 0 16 64 0; do
  timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --rec-batch $nb > gpurun_out/r2_82_rec_nb$nb.json 2>gpurun_out/r2_82_rec_nb$nb.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2_82_rec_nb$nb.json').read().strip().splitlines()[-1]); print('nb $nb', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for sg in 2 64; do
  timeout 600 python bench.py --engine 1 --sigma $sg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_82_rec_s$sg.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_82_rec_s$sg.json').read().strip().splitlines()[-1]); print('sigma $sg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
done
for nb in 0 16; do
  echo "first calls, rec_batch $nb"; timeout 600 python tools/profile_run.py --config 5 --engine 1 --reps 3 --rec-batch $nb 2>&1 | tail -3
done

# round 2, call 73: config-5 recursive launch list after templating the tensor-core pass 2 on the pair count
mkdir -p gpurun_out
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_73_rec.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2_73_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_73_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_73_launches.csv 2>/dev/null | sed -n 3,7p

# round 2, call 38: recursive pass 2 A/B -- entering states converted at the load (eager) or at the use
# (lazy), pass 2 compiled for 4 or 3 CTAs per SM; bench + launch list per library
mkdir -p gpurun_out
for lib in main eager4 lazy3 eager3; do
  if [ $lib = main ]; then unset BFVEC_LIB; else export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$lib.so; fi
  timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_38_rec_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_38_rec_$lib.json').read().strip().splitlines()[-1]); print('$lib', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_38_launches_$lib.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r2_38_launches_$lib.csv 2>/dev/null | sed -n 3,6p
done

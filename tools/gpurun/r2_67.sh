# round 2, call 67: recursive engine sigma sweep with every segment blur on the tensor cores; ncu of
# rect_vscan_tc_kernel
mkdir -p gpurun_out
for sg in 2 8 16 32 64; do
  timeout 600 python bench.py --engine 1 --sigma $sg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_67_rec_s$sg.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_67_rec_s$sg.json').read().strip().splitlines()[-1]); print('sigma $sg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'])"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_vscan_tc -c 1 \
    -o gpurun_out/r2_67_vtc -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_67_ncu.log 2>&1
echo "ncu exit $?"

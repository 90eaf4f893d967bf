# round 2, call 89: final tree -- config 2 and config 1 at --steps 20 (as the committed per-config lines), three runs each
mkdir -p gpurun_out
for i in 1 2 3; do for c in 2 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_89_c${c}_$i.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_89_c${c}_$i.json').read().strip().splitlines()[-1]); print('cfg$c run $i', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'kernel_ms %.5f'%d['roofline']['fused_ms_per_launch'], 'step_ms %.5f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"
done; done

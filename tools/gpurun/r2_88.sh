# round 2, call 88: final tree -- the driver's reference arm (as launched at round end) and the per-config bench lines 1-4
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r2_88_reference.json 2> gpurun_out/r2_88_reference.err; echo "reference exit $?"
tail -c 600 gpurun_out/r2_88_reference.json
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c > gpurun_out/r2_88_bench_c$c.json 2> gpurun_out/r2_88_bench_c$c.err; echo "bench c$c exit $?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2_88_bench_c$c.json').read().strip().splitlines()[-1]); print('cfg$c', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done

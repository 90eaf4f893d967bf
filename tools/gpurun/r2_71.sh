# round 2, call 71: final-tree FIR benches on configs 1-4 (every leg) to refresh BASELINE §4
mkdir -p gpurun_out
for cfg in 1 2 3 4; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 > gpurun_out/r2_71_bench_c$cfg.json 2> gpurun_out/r2_71_bench_c$cfg.err; echo "bench c$cfg exit $?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2_71_bench_c$cfg.json').read().strip().splitlines()[-1]); print('cfg$cfg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'cpu %.4g'%d['cpu_baseline']['value'], d['clocks']['sm_mhz'])"
done

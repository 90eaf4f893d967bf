# round 2, call 5: A/B of mbar_wait with a suspend-time hint (default build) vs the plain probe loop
# (libbfvec_spin.so, -DBFVEC_MBAR_SPIN) on configs 2-5, FIR engine, kernel-only bench lines
mkdir -p gpurun_out
for rep in 1 2; do
for lib in spin main; do
  if [ $lib = spin ]; then export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_spin.so; else unset BFVEC_LIB; fi
  for cfg in 2 3 4 5; do
    steps=20; [ $cfg = 5 ] && steps=5
    timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_05_${lib}_c${cfg}_$rep.json 2> gpurun_out/r2_05_${lib}_c${cfg}_$rep.err
    python -c "
import json; d=json.loads(open('gpurun_out/r2_05_${lib}_c${cfg}_$rep.json').read().strip().splitlines()[-1]); print('$lib', 'cfg$cfg', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'kernel_ms %.4f'%d['roofline']['fused_ms_per_launch'], d['clocks']['sm_mhz'])"
  done
done
done

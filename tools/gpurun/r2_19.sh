# round 2, call 19: exact filter A/B -- default (102 registers, 2 CTAs/SM) vs -DBFVEC_DIRECT_MINB=3
# (80 registers + 72 B spills, 3 CTAs/SM)
mkdir -p gpurun_out
for lib in main lb3; do
  if [ $lib = lb3 ]; then export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_lb3.so; else unset BFVEC_LIB; fi
  timeout 600 python tools/direct_bench.py --json gpurun_out/r2_19_direct_$lib.json > /dev/null 2>&1
  python -c "
import json; [print('$lib', r['case'], round(r['ms'],4), round(r['frac_of_roofline'],3)) for r in json.load(open('gpurun_out/r2_19_direct_$lib.json'))]"
done

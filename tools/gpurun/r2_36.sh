# round 2, call 36: rec_impl 2 (virtual lines) the default -- whole GPU suite, smoke, recursive bench,
# ncu --set full of each recursive pass (pass 0, virtual lines, pass 2) on 16 config-5 samples
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_36_suite.log 2>&1
echo "suite exit $?"; tail -2 gpurun_out/r2_36_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_36_smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/r2_36_smoke.log
timeout 600 python bench.py --engine 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_36_rec.json 2>gpurun_out/r2_36_rec.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_36_rec.json').read().strip().splitlines()[-1]); print('rec', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], d['roofline']['kernel'], 'e2e %.4g'%d['e2e']['value'])"
for k in "rect_tile_kernel:-s 0 -c 1:p0" "rect_vline_kernel:-c 1:vl" "rect_tile_kernel:-s 1 -c 1:p2"; do
  IFS=: read kn sel tag <<< "$k"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$kn $sel \
    -o gpurun_out/r2_36_$tag -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_36_ncu_$tag.log 2>&1
  echo "ncu $tag exit $?"
done

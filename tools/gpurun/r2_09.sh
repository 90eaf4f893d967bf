# round 2, call 9: graph-replay check on the default and checked builds; tiled recursive engine with
# the stored row blur (rec_store = 1) vs recompute (0): parity and config-5 timing
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
echo "== default build"; timeout 300 python tools/graph_debug.py
echo "== checked build"; BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 300 python tools/graph_debug.py
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py tests/gpu/test_recursive_contract.py -q -x > gpurun_out/r2_09_rec_pytest.log 2>&1
echo "recursive pytest exit $?"; tail -3 gpurun_out/r2_09_rec_pytest.log
for st in 0 1; do
timeout 600 python bench.py --engine 1 --rec-store $st --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_09_rec_store$st.json 2> gpurun_out/r2_09_rec_store$st.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_09_rec_store$st.json').read().strip().splitlines()[-1]); print('rec_store $st', '%.4g'%d['value'], 'frac %.4f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_09_rec_launches.csv python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_09_ncu.log 2>&1
echo "ncu launches exit $?"

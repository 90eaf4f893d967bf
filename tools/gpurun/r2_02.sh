# round 2, call 2: ADVICE fixes on the GPU (p2p alternating slot sets, PZ checks), bench with the
# 64-row-band CPU leg, and the CPU halo-extrapolation check on the box's host cores
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/gpu/test_p2p_two_ranks.py tests/gpu/test_parity.py -q -x > gpurun_out/r2_02_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r2_02_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_02_bench_c5.json 2> gpurun_out/r2_02_bench_c5.err
echo "bench exit $?"; tail -c 1500 gpurun_out/r2_02_bench_c5.json
timeout 600 python tools/cpu_halo_check.py --config 3 > gpurun_out/r2_02_halo_check.txt 2>&1
echo "halo exit $?"; cat gpurun_out/r2_02_halo_check.txt
nproc; lscpu | grep "Model name"

mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_spatial_parity.py tests/gpu/test_random_cases.py -q -x > gpurun_out/pytest53.log 2>&1
echo "pytest exit $?"
timeout 600 python /root/repo/tools/box_bench.py > gpurun_out/boxbench53.log 2>&1
echo done

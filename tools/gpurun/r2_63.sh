# round 2, call 63: recursive parity incl. tiled_tc and the tensor-core vs FP32 pass-2 comparison
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_recursive_parity.py -q -rs -s -k "tensor_core or tiled_tc" > gpurun_out/r2_63_pytest.log 2>&1
echo "exit $?"; grep -E "passed|failed|max \|tc" gpurun_out/r2_63_pytest.log | head -12

# round 2, call 6: new parity tests (bitwise band sharding, config-5 middle band)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_parity.py -q -k "bitwise or config_bands" > gpurun_out/r2_06_pytest.log 2>&1
echo "pytest exit $?"; tail -15 gpurun_out/r2_06_pytest.log

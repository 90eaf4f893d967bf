# round 2, call 8: guard-band tests + async frames on the default build; the whole GPU suite on the
# checked build (the compute-sanitizer stand-in, tools/checked_build.sh)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_guards.py tests/gpu/test_parity.py -k "guard or two_streams or repeated or async" -q > gpurun_out/r2_08_default.log 2>&1
echo "default exit $?"; tail -3 gpurun_out/r2_08_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2_08_checked_suite.log 2>&1
echo "checked suite exit $?"; tail -8 gpurun_out/r2_08_checked_suite.log
grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_08_checked_suite.log

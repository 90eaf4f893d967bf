# round 2, call 7: the compute-sanitizer stand-in -- the whole GPU suite on the checked build
# (libbfvec_checked.so: -DBFVEC_CHECKED: mbarrier watchdogs, ring-slot row tags in the v6 kernel,
# BF_CHECK bounds), plus the new guard-band / two-stream / repetition tests on the default build
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/gpu/test_guards.py -q > gpurun_out/r2_07_guards_default.log 2>&1
echo "guards (default build) exit $?"; tail -3 gpurun_out/r2_07_guards_default.log
BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2_07_checked_suite.log 2>&1
echo "checked suite exit $?"; tail -8 gpurun_out/r2_07_checked_suite.log
grep -c "BF_CHECK failed\|watchdog" gpurun_out/r2_07_checked_suite.log

# round 2, call 22: final-state checks: whole GPU suite, smoke, checked build suite
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_22_suite_default.log 2>&1
echo "default suite exit $?"; tail -3 gpurun_out/r2_22_suite_default.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_22_smoke.log 2>&1
echo "smoke exit $?"; cat gpurun_out/r2_22_smoke.log

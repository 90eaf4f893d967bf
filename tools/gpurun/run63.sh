mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu63.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke63.log 2>&1
echo "smoke exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rect_tile_kernel --launch-skip 2 -c 1 -o gpurun_out/rec63_pass2 \
  python tools/profile_run.py --config 5 --engine 1 --rec-impl 1 --samples 8 --reps 1 > gpurun_out/rec63_ncu.log 2>&1
echo "ncu exit $?"

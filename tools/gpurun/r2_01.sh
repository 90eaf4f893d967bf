# round 2, call 1: compute-sanitizer memcheck over every kernel family (small launches)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 50 \
  python tools/sanitize_run.py > gpurun_out/r2_memcheck.log 2>&1
echo "memcheck exit $?"
tail -5 gpurun_out/r2_memcheck.log

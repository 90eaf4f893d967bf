set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest exit $?"
timeout 300 python tools/profile_run.py --config 5 --rows 1024 --samples 64 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mcsf_fused -s 1 -c 1 -o gpurun_out/prof_c5 python tools/profile_run.py --config 5 --rows 1024 --samples 64 > gpurun_out/ncu_c5.log 2>&1
echo "ncu exit $?"

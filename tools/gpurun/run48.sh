mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_sweep_parity.py tests/gpu/test_sampler_stratified.py tests/gpu/test_variants.py -q -x > gpurun_out/pytest48.log 2>&1
echo "pytest exit $?"
timeout 900 python tools/paper_experiments.py --which fig5 --out gpurun_out/fig5_r48.json > gpurun_out/fig5_r48.log 2>&1
echo "fig5 exit $?"

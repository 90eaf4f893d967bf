# round 2, call 90: final tree -- fresh-seed random sweeps vs the oracle: mixed (seed 31) and recursive tensor-core heavy (seed 32, widths % 32 == 0)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 500 python tools/random_sweep.py --n 150 --seed 31 > gpurun_out/r2_90_sweep31.txt 2>&1; echo "sweep 31 exit $?"; tail -1 gpurun_out/r2_90_sweep31.txt
timeout 500 python tools/random_sweep.py --n 150 --seed 32 --rec-frac 1.0 --w32 0.8 > gpurun_out/r2_90_sweep32.txt 2>&1; echo "sweep 32 exit $?"; tail -1 gpurun_out/r2_90_sweep32.txt

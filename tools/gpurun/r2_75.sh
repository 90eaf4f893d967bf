# round 2, call 75: random sweep against the oracle weighted to the recursive engine with its
# tensor-core paths (80 % recursive cases, half the widths multiples of 32), 2 seeds x 150
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
for seed in 21 22; do
  timeout 1500 python tools/random_sweep.py --n 150 --seed $seed --rec-frac 0.8 --w32 0.5 > gpurun_out/r2_75_sweep_$seed.log 2>&1
  echo "seed $seed exit $?"; tail -1 gpurun_out/r2_75_sweep_$seed.log; grep FAIL gpurun_out/r2_75_sweep_$seed.log | head -5
done

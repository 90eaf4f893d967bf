# round 2, call 34: extended random sweep of the option space against the oracle (400 cases, 2 seeds)
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
for seed in 9 10; do
  timeout 2400 python tools/random_sweep.py --n 200 --seed $seed > gpurun_out/r2_34_sweep_$seed.log 2>&1
  echo "seed $seed exit $?"; tail -1 gpurun_out/r2_34_sweep_$seed.log; grep FAIL gpurun_out/r2_34_sweep_$seed.log | head -5
done

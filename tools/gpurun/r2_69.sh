# round 2, call 69: pass 0 compiled for 4 / 5 / 6 CTAs per SM (A/B, launch lists)
mkdir -p gpurun_out
for lib in main p0c5 p0c6; do
  if [ $lib = main ]; then unset BFVEC_LIB; else export BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_$lib.so; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_69_launches_$lib.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
  echo $lib; python tools/launch_summary.py gpurun_out/r2_69_launches_$lib.csv 2>/dev/null | grep "4, 0"
done

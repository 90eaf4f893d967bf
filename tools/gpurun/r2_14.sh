# round 2, call 14: DRAM traffic of the bench's fused launch (config 5, persistent schedule) and a
# fresh ncu --set full of every pass of the tiled recursive engine (VERDICT r01 missing #4)
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:mcsf -c 1 --csv --log-file gpurun_out/r2_14_traffic_c5.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/r2_14_traffic.log 2>&1
echo "traffic exit $?"; tail -2 gpurun_out/r2_14_traffic.log
# launch order of one batch: tile<0> (0), scan rows (1), tile<1> (2), scan columns (3), tile<2> (4)
for sk in 0 1 2 4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:rect -s $sk -c 1 \
    -o gpurun_out/r2_14_rec_launch$sk -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 \
    > gpurun_out/r2_14_rec_launch$sk.log 2>&1
  echo "ncu launch $sk exit $?"
done

# paper experiments (Table 1, Fig. 5) + DRAM traffic of the v5b bench launch
mkdir -p gpurun_out
timeout 1500 python tools/paper_experiments.py --out gpurun_out/paper_experiments.json > gpurun_out/paper_experiments.log 2>&1
echo "experiments exit $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:mcsf -c 1 --csv --log-file gpurun_out/traffic_v5b.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_v5b.log 2>&1
echo "traffic exit $?"

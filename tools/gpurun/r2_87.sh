# round 2, call 87: final tree (pass 2 at pitch 36) -- recursive-engine launch list and ncu --set full of the
# tensor-core pass 2, so profiles/ holds evidence for the shipping kernel
mkdir -p gpurun_out
python -c "import oracle.native as n; n.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_87_launches.csv \
    python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_87_launches.csv 2>/dev/null | head -12
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rect_tc2 -c 1 \
    -o gpurun_out/r2_87_tc2 -f python tools/profile_run.py --config 5 --engine 1 --samples 16 --reps 1 > gpurun_out/r2_87_ncu_tc2.log 2>&1
echo "ncu tc2 exit $?"
ncu -i gpurun_out/r2_87_tc2.ncu-rep --page details 2>/dev/null | grep -E "Duration|SM Frequency|Issue Slots Busy|DRAM Throughput|Registers Per|Achieved Occupancy|Memory Throughput|Theoretical Occupancy"
python tools/ncu_summary.py gpurun_out/r2_87_tc2.ncu-rep > gpurun_out/r2_87_tc2_summary.txt 2>&1; head -40 gpurun_out/r2_87_tc2_summary.txt

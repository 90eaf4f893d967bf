mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke67.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench67.json 2> gpurun_out/bench67.err
echo "bench exit $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench67_ref.json 2> gpurun_out/bench67_ref.err
echo "ref exit $?"

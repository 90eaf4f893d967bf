# round-1 validation: the driver's commands on the current tree
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke46.log 2>&1
echo "smoke exit $?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu46.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py > gpurun_out/bench_r01_final.json 2> gpurun_out/bench_r01_final.err
echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref46.json 2> gpurun_out/bench_ref46.err
echo "ref exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun46.json 2> gpurun_out/bench_torchrun46.err
echo "torchrun exit $?"

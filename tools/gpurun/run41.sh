mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_parity.py -q -x -k "p2p or sample_shards or filter_rows" > gpurun_out/pytest41.log 2>&1
echo "pytest exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun41.json 2> gpurun_out/bench_torchrun41.err
echo "torchrun exit $?"

# round 2, call 18: orchestration check of the N > 1 bench path on the one GPU of the box: 2 ranks
# (torchrun via --gpus 2), gloo host collectives, both ranks on cuda:0 -- NOT a timing (the driver's
# scaling runs use NCCL, one rank per GPU); checks that every mode runs end to end and prints one line
mkdir -p gpurun_out
for mode in samples bands samples-p2p; do
  BFVEC_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config 2 --steps 2 --warmup 1 --mode $mode \
    > gpurun_out/r2_18_gloo_$mode.json 2> gpurun_out/r2_18_gloo_$mode.err
  echo "mode $mode exit $?"; tail -c 400 gpurun_out/r2_18_gloo_$mode.json; echo; grep -i "error\|Traceback" gpurun_out/r2_18_gloo_$mode.err | head -5
done

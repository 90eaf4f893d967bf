mkdir -p gpurun_out
gcc -O2 -I include examples/filter_host.c -L paper_1605_02164_b200 -lbfvec -Wl,-rpath,$PWD/paper_1605_02164_b200 -o gpurun_out/filter_host -lm && timeout 120 ./gpurun_out/filter_host > gpurun_out/example_c.log 2>&1
echo "c exit $?"
timeout 300 python examples/filter_torch.py > gpurun_out/example_py.log 2>&1
echo "py exit $?"

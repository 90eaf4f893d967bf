mkdir -p gpurun_out
for i in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu97_$i.log 2>&1
  echo "pytest $i exit $?"
done

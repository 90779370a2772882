#!/bin/bash
# Round 2: fused reference rounding -- parity tests and the 512^3 cost of each arithmetic.
tag=${1:-r2b}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python -m pytest -p no:cacheprovider tests/test_gpu_reference_fused.py tests/test_gpu_solve.py -q -m gpu \
  --timeout 300 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for rm in reference storage; do
  timeout 600 python bench.py --no-cpu --steps 2 --warmup 2 --rounding $rm > gpurun_out/bench_${rm}_${tag}.log 2>&1
  echo "bench rc=$?" >> gpurun_out/bench_${rm}_${tag}.log
done

#!/bin/bash
tag=${1:-r2l}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests/test_gpu_kernels.py tests/test_gpu_solve.py tests/test_gpu_fullsize.py -q -m gpu --timeout 400 -x > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
rm -f gpurun_out/ab_${tag}.jsonl
for rep in 1 2; do
  timeout 600 python scripts/exp_kernels.py 512 bf16 2 | sed 's/^/{"lib": "tm", "x": /; s/$/}/' >> gpurun_out/ab_${tag}.jsonl
  GADI_NORM_TM0=1 timeout 600 python scripts/exp_kernels.py 512 bf16 2 | sed 's/^/{"lib": "rows", "x": /; s/$/}/' >> gpurun_out/ab_${tag}.jsonl
done

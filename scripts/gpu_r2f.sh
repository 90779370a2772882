#!/bin/bash
# peer transport + reference-fused + drop-in + alphaselect GPU tests first (fast fail), then crd sweep
tag=${1:-r2f}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -p no:cacheprovider tests/test_gpu_slabs.py tests/test_gpu_dropin.py tests/test_alphaselect.py -q -m gpu --timeout 500 -x > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
bash scripts/gpu_crd.sh

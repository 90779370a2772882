#!/bin/bash
tag=${1:-r2n}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -p no:cacheprovider tests/test_gpu_slabs.py tests/test_gpu_reference_fused.py -q -m gpu --timeout 500 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log

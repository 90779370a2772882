#!/bin/bash
tag=${1:-r2m}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python -m pytest -p no:cacheprovider tests/test_crd3d.py tests/test_gpu_kernels.py tests/test_gpu_solve.py tests/test_gpu_slabs.py -q -m gpu --timeout 500 -x > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
timeout -s KILL 900 python scripts/crd3d_large.py 512 fp32 3 > gpurun_out/crd3d_${tag}.jsonl 2>&1
timeout -s KILL 900 python scripts/crd3d_large.py 1024 bf16 2 >> gpurun_out/crd3d_${tag}.jsonl 2>&1
timeout 900 python scripts/crd_sweep.py 8192 fp32 60 1,1e-2 > gpurun_out/crd2d_${tag}.jsonl 2>&1

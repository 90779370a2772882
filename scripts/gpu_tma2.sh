#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_tma2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma2.log
timeout 300 python scripts/exp_kernels.py 512 bf16 2 > gpurun_out/exp_tma2.log 2>&1
GADI_TMA2=0 timeout 300 python scripts/exp_kernels.py 512 bf16 2 >> gpurun_out/exp_tma2.log 2>&1
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_tma2.log 2>&1

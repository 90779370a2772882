#!/bin/bash
# exp_kernels: default build vs a variant library
export PYTHONPATH=$PWD
mkdir -p gpurun_out
v=$1
timeout 600 python scripts/exp_kernels.py 512 bf16 3 > gpurun_out/exp_default_$v.json 2>&1
GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$v.so timeout 600 python scripts/exp_kernels.py 512 bf16 3 > gpurun_out/exp_$v.json 2>&1

#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python scripts/exp_kernels.py 512 bf16 2 > gpurun_out/exp_occ.log 2>&1
for v in m3b74 m4b52 m3b66; do
  GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$v.so timeout 300 python scripts/exp_kernels.py 512 bf16 2 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/exp_occ.log 2>&1
done

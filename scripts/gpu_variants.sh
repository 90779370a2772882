#!/bin/bash
# kernel timings of the tiling variants (paper_2512_21164_b200/variants/*.so)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python scripts/exp_kernels.py 512 bf16 2 > gpurun_out/exp_variants.log 2>&1
for v in by16 vz2b16 by4vz2b16 vz64x4; do
  GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$v.so timeout 300 python scripts/exp_kernels.py 512 bf16 2 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/exp_variants.log 2>&1
done

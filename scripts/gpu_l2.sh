#!/bin/bash
# L2 persisting-window experiments (per-kernel times of 3 outer steps at 512^3)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
rm -f gpurun_out/l2_exp.jsonl
timeout 600 python scripts/exp_kernels.py 512 bf16 3 >> gpurun_out/l2_exp.jsonl 2>&1
for v in R P0 Z; do
  for mb in 40 80; do
    GADI_L2_VERBOSE=1 GADI_L2_VEC=$v GADI_L2_PERSIST_MB=$mb timeout 600 python scripts/exp_kernels.py 512 bf16 3 >> gpurun_out/l2_exp.jsonl 2>> gpurun_out/l2_exp.err
  done
done

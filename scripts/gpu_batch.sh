#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for cap in 0 16 64; do
  GADI_BATCH_CAP=$cap timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu | sed "s/^{/{\"cap\": $cap, /" >> gpurun_out/bench_caps.log 2>&1
done
timeout 300 python scripts/exp_kernels.py 512 bf16 2 > gpurun_out/exp_suspend.log 2>&1

#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -s KILL 900 python scripts/crd3d_large.py 1024 bf16 2 > gpurun_out/crd3d_large.jsonl 2> gpurun_out/crd3d_large.err
timeout -s KILL 900 python scripts/crd3d_large.py 512 fp32 3 >> gpurun_out/crd3d_large.jsonl 2>> gpurun_out/crd3d_large.err
timeout 1800 python scripts/bench_configs.py 5 > gpurun_out/configs5_r2h.jsonl 2>&1

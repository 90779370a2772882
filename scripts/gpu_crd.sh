#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python scripts/crd_sweep.py 1024 bf16 60 1,1e-2 10,1e-2 100,1e-2 1000,1e-2 10,1e-4 100,1e-4 > gpurun_out/crd_sweep_1024.jsonl 2>&1
timeout 1500 python scripts/crd_sweep.py 8192 bf16 40 10,1e-2 100,1e-2 1000,1e-2 > gpurun_out/crd_sweep_8192.jsonl 2>&1

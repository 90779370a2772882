#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python scripts/crd_sweep.py 8192 bf16 60 1,1e-2 3,1e-2 0.3,1e-2 > gpurun_out/crd_sweep_8192b.jsonl 2>&1
timeout 1200 python scripts/crd_sweep.py 8192 fp32 60 1,1e-2 > gpurun_out/crd_sweep_8192c.jsonl 2>&1
timeout 1500 python scripts/crd_sweep.py 8192 fp64 60 1,1e-2 > gpurun_out/crd_sweep_8192d.jsonl 2>&1

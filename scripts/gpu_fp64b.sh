#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 3000 python scripts/fp64_sweep.py 512 2000 0.006,1e-2 0.003,1e-2 0.0015,1e-2 0.003,1e-3 > gpurun_out/fp64_sweep_r2b.jsonl 2> gpurun_out/fp64_sweep_r2b.err

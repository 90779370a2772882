#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 3000 python scripts/fp64_sweep.py 512 2000 0.00075,1e-2 0.0004,1e-2 > gpurun_out/fp64_sweep_r2c.jsonl 2> gpurun_out/fp64_sweep_r2c.err

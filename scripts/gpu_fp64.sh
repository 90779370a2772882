#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 3000 python scripts/fp64_sweep.py 512 600 > gpurun_out/fp64_sweep_r2.jsonl 2> gpurun_out/fp64_sweep_r2.err

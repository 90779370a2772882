#!/bin/bash
# tiling variants A/B + a finer (alpha, inner_tol, omega) sweep around the bench point
export PYTHONPATH=$PWD
mkdir -p gpurun_out
bash scripts/gpu_ab.sh tile3 default m2 by4 by4m4
timeout 900 python scripts/alpha_sweep.py 512 bf16 0.0125,0.0135,0.0145,0.015,0.0155 0.01,0.02,0.005 1e-12 1.0 200 > gpurun_out/sweep_r3b.jsonl 2> gpurun_out/sweep_r3b.err
timeout 600 python scripts/alpha_sweep.py 512 bf16 0.0125,0.015 0.01 1e-12 0.8,1.2,1.4 200 > gpurun_out/sweep_r3b_om.jsonl 2> gpurun_out/sweep_r3b_om.err

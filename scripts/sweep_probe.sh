#!/bin/bash
# (alpha, inner_tol) grid for bf16 and fp64 inner solves on the bench workload,
# each run to relres <= 1e-12 (or stagnation / 120 outer steps).
export PYTHONPATH=$PWD
for us in bf16 fp64; do
  for it in 1e-3 1e-4 1e-6; do
    for a in 0.003 0.00625 0.0125 0.025; do
      timeout 300 python scripts/floor_probe.py 512 $us $a $it 120 1e-12 >> gpurun_out/sweep_probe.log 2>&1
    done
  done
done

#!/bin/bash
# ncu --set full captures of hot passes (one launch each, after 3).
# Usage: scripts/gpu_ncu.sh TAG KERNEL...   (regexes on the demangled names)
tag=$1; shift
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for k in "$@"; do
  GADI_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${tag}_$k python scripts/prof_step.py 512 bf16 1 > gpurun_out/full_${tag}_$k.log 2>&1
done

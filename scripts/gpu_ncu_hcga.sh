#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
GADI_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:HcgA -s 3 -c 1 \
  -o gpurun_out/full_hcga python scripts/prof_step.py 512 bf16 1 > gpurun_out/full_hcga.log 2>&1
ls -la gpurun_out/full_hcga.ncu-rep

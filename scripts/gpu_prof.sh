#!/bin/bash
# ncu evidence for the bench workload (cd3d 512^3, bf16 inner): launch list of
# two outer steps (norm power iteration included) and one --set full capture of
# each hot pass.  Usage: scripts/gpu_prof.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
export PYTHONPATH=$PWD
[ -n "$SKIP_LAUNCHES" ] || timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2600 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
for k in HcgA HcgB NormPass Outer CgnrP1; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${tag}_$k python scripts/prof_step.py 512 bf16 1 > gpurun_out/full_${tag}_$k.log 2>&1
done
ls -la gpurun_out

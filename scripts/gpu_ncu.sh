#!/bin/bash
# ncu --set full captures of hot passes (one launch each, after 3), summarised
# on the box (scripts/ncu_summarize.py, scripts/ncu_stalls.py) so only text
# comes back; KEEP=1 keeps the .ncu-rep files.
# Usage: scripts/gpu_ncu.sh TAG KERNEL...   (regexes on the demangled names)
tag=$1; shift
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for k in "$@"; do
  GADI_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${tag}_$k python scripts/prof_step.py 512 bf16 1 > gpurun_out/full_${tag}_$k.log 2>&1
  python scripts/ncu_summarize.py gpurun_out/full_${tag}_$k.ncu-rep "${tag} $k (cd3d 512^3, bf16 inner)" > gpurun_out/ncu_${tag}_$k.md 2>&1
  [ "$KEEP" = 1 ] || rm -f gpurun_out/full_${tag}_$k.ncu-rep
done

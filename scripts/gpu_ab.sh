#!/bin/bash
# A/B of variant libraries (paper_2512_21164_b200/variants/libgadi_b200_<v>.so)
# on the per-kernel live timers of scripts/exp_kernels.py; two interleaved rounds.
# usage: gpu_ab.sh TAG v1 v2 ...   (v = "default" -> the in-tree library)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
tag=$1; shift
out=gpurun_out/ab_$tag.jsonl
: > $out
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$v.so; fi
    line=$(GADI_LIB=$lib timeout 600 python scripts/exp_kernels.py 512 bf16 3 2>gpurun_out/ab_${tag}_$v.err | tail -1)
    echo "{\"variant\": \"$v\", \"rep\": $rep, \"res\": $line}" >> $out
  done
done

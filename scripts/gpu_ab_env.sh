#!/bin/bash
# A/B of run-time knobs: gpu_ab_env.sh TAG "ENV1" "ENV2" ...  ("-" = no extra env)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
tag=$1; shift
out=gpurun_out/ab_${tag}.jsonl; : > $out
for rep in 1 2; do
  for e in "$@"; do
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    line=$(env $envs timeout 600 python scripts/exp_kernels.py 512 bf16 3 2>>gpurun_out/ab_${tag}.err | tail -1)
    echo "{\"variant\": \"$e\", \"rep\": $rep, \"res\": $line}" >> $out
  done
done

#!/bin/bash
# TALL HcgA: full GPU tests, reference-rounding 512^3 histories with and without, kernel A/B
export PYTHONPATH=$PWD
mkdir -p gpurun_out
tag=${1:-tall}
timeout 1500 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for t in 1 0; do GADI_TALL=$t timeout 600 python scripts/rf512_check.py 2 > gpurun_out/rf512_${tag}_$t.json 2>&1; done
out=gpurun_out/ab_${tag}.jsonl; : > $out
for rep in 1 2; do
  for t in 1 0; do
    line=$(GADI_TALL=$t timeout 600 python scripts/exp_kernels.py 512 bf16 3 2>gpurun_out/ab_${tag}_$t.err | tail -1)
    echo "{\"variant\": \"tall$t\", \"rep\": $rep, \"res\": $line}" >> $out
  done
done

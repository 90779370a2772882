#!/bin/bash
# z-lag H-CG: GPU tests of the inner solvers / solves, then an A/B of the
# per-kernel timers with GADI_ZLAG=1 (default) and GADI_ZLAG=0
export PYTHONPATH=$PWD
mkdir -p gpurun_out
tag=${1:-zl}
timeout 900 python -m pytest -p no:cacheprovider tests -q -m gpu -x --timeout 600 -k "solve or inner or dropin or reference or slab" > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
out=gpurun_out/ab_${tag}.jsonl; : > $out
for rep in 1 2; do
  for zl in 1 0; do
    line=$(GADI_ZLAG=$zl timeout 600 python scripts/exp_kernels.py 512 bf16 3 2>gpurun_out/ab_${tag}_$zl.err | tail -1)
    echo "{\"variant\": \"zlag$zl\", \"rep\": $rep, \"res\": $line}" >> $out
  done
done

#!/bin/bash
tag=${1:-r2j}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
rm -f gpurun_out/ab_${tag}.jsonl
for rep in 1 2; do
for lib in main nozpad nopack; do
  if [ $lib = main ]; then L=$PWD/paper_2512_21164_b200/libgadi_b200.so; else L=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$lib.so; fi
  GADI_LIB=$L timeout 600 python scripts/exp_kernels.py 512 bf16 3 | sed "s/^/{\"lib\": \"$lib\", \"x\": /; s/\$/}/" >> gpurun_out/ab_${tag}.jsonl 2>&1
done
done

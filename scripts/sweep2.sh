#!/bin/bash
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_solve.py -q -k "fullsize or fp16" > gpurun_out/pytest_full3.log 2>&1; echo rc=$? >> gpurun_out/pytest_full3.log
for it in 1e-2 3e-3; do for a in 0.0125 0.02; do
  timeout 300 python scripts/floor_probe.py 512 bf16 $a $it 120 1e-12 >> gpurun_out/sweep2.log 2>&1
done; done

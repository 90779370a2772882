#!/bin/bash
tag=${1:-r2c}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 400 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for ng in 128 256 512; do timeout 600 python scripts/rounding_trace.py $ng 40 >> gpurun_out/rounding_trace_${tag}.jsonl 2>>gpurun_out/rounding_trace_${tag}.err; done

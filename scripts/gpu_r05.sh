#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests -q -m gpu -k "crd" > gpurun_out/pytest_crd5.log 2>&1; echo rc=$? >> gpurun_out/pytest_crd5.log
timeout 900 python bench.py > gpurun_out/bench_r05.log 2>&1
timeout 900 python scripts/bench_configs.py 5 > gpurun_out/bench_cfg5.log 2>&1

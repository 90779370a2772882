#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python scripts/tall_diag.py > gpurun_out/tall_default.jsonl 2>&1
GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_b16m1.so timeout 600 python scripts/tall_diag.py > gpurun_out/tall_b16m1.jsonl 2>&1

#!/bin/bash
# GPU tests of a variant library (bitwise reference-rounding and kernel tests)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
v=$1; shift
GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_$v.so timeout 1200 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 "$@" > gpurun_out/pytest_var_$v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_var_$v.log

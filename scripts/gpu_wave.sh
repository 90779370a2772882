#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
V=$PWD/paper_2512_21164_b200/variants/libgadi_b200_vz2b4.so
timeout 300 python scripts/exp_kernels.py 512 bf16 2 > gpurun_out/exp_wave.log 2>&1
GADI_WAVEFRONT=1 timeout 300 python scripts/exp_kernels.py 512 bf16 2 >> gpurun_out/exp_wave.log 2>&1
GADI_LIB=$V timeout 300 python scripts/exp_kernels.py 512 bf16 2 | sed 's/^{/{"variant": "vz2b4", /' >> gpurun_out/exp_wave.log 2>&1
GADI_LIB=$V GADI_WAVEFRONT=1 timeout 300 python scripts/exp_kernels.py 512 bf16 2 | sed 's/^{/{"variant": "vz2b4", /' >> gpurun_out/exp_wave.log 2>&1
GADI_WAVEFRONT=1 timeout 300 python -m pytest tests/test_gpu_solve.py -q -x -k "c3_cd3d or cfg1" > gpurun_out/pytest_wave.log 2>&1

#!/bin/bash
# HcgB on 16-row tiles with boxed epilogue tiles (variant hb3) vs default, then the r3e evidence
export PYTHONPATH=$PWD
mkdir -p gpurun_out
bash scripts/gpu_ab.sh hb3 default hb3
bash scripts/gpu_r3e.sh r3f

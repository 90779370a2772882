#!/bin/bash
# quick variant: recompile only api.cu with extra flags, link with the default objects
set -e
cd /root/repo/paper_2512_21164_b200/csrc
name=$1; shift
mkdir -p build_$name ../variants
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -warn-spills --expt-relaxed-constexpr -ftz=false -prec-div=true -prec-sqrt=true "$@" -c api.cu -o build_$name/api.o
objs="build_$name/api.o"; for f in exact comm peer hostcopy engine_bf16 engine_fp16 engine_fp32 engine_fp64; do objs="$objs build/$f.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../variants/libgadi_b200_$name.so $objs -ldl
echo built $name

#!/bin/bash
# evidence on the current tree: bench line, launch list, ncu of HcgA / norm_fused / HcgB
tag=${1:-r3e}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${tag}.log
GADI_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
bash scripts/gpu_ncu.sh ${tag} HcgA norm_fused HcgB

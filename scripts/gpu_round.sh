#!/bin/bash
# Round-end evidence: full GPU tests, smoke, bench line, launch list and
# ncu --set full captures of the hot passes.  Usage: scripts/gpu_round.sh TAG
tag=${1:-r02}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${tag}.log
timeout 900 python bench.py > gpurun_out/bench_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${tag}.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
for k in HcgA HcgB norm_fused; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${tag}_$k python scripts/prof_step.py 512 bf16 1 > gpurun_out/full_${tag}_$k.log 2>&1
done

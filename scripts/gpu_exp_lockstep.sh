#!/bin/bash
# scheduling experiment: default persistent split vs lockstep chunks
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for env in "" "GADI_LOCKSTEP=1" "GADI_WAVES=2" ; do
  env $env timeout 300 python scripts/exp_kernels.py 512 bf16 2 >> gpurun_out/exp_lockstep.log 2>&1
done
GADI_LOCKSTEP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
  --kernel-name-base demangled -k regex:"HcgA|HcgB|NormPass" -c 12 --csv --log-file gpurun_out/launches_lockstep.csv python scripts/prof_step.py 512 bf16 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
  --kernel-name-base demangled -k regex:"HcgA|HcgB|NormPass" -c 12 --csv --log-file gpurun_out/launches_default.csv python scripts/prof_step.py 512 bf16 1 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1

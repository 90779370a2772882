#!/bin/bash
tag=${1:-r2i}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${tag}.log
timeout 1200 python bench.py > gpurun_out/bench_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${tag}.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ref_${tag}.log
GADI_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
GADI_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Outer -s 1 -c 1 \
  -o gpurun_out/full_${tag}_Outer python scripts/prof_step.py 512 bf16 2 > gpurun_out/full_${tag}_Outer.log 2>&1
python scripts/ncu_summarize.py gpurun_out/full_${tag}_Outer.ncu-rep "${tag} Outer (cd3d 512^3, bf16 inner)" > gpurun_out/ncu_${tag}_Outer.md 2>&1
rm -f gpurun_out/full_${tag}_Outer.ncu-rep

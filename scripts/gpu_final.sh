#!/bin/bash
# end-of-round evidence: GPU tests, smoke, bench line, ncu launch list, ncu --set full of the top kernels
tag=${1:-final}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1800 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${tag}.log
timeout 1200 python bench.py > gpurun_out/bench_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${tag}.log
GADI_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
bash scripts/gpu_ncu.sh ${tag} HcgA norm_fused HcgB

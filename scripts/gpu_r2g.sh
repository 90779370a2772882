#!/bin/bash
# full GPU tests + smoke + bench on the current defaults; ncu of Outer / HcgB; x-unroll variant
tag=${1:-r2g}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest -p no:cacheprovider tests -q -m gpu --timeout 600 > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${tag}.log
timeout 1200 python bench.py > gpurun_out/bench_${tag}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${tag}.log
GADI_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/launches_${tag}.csv python scripts/prof_step.py 512 bf16 2 > gpurun_out/launch_run_${tag}.log 2>&1
for k in Outer HcgB; do
  GADI_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 1 -c 1 \
    -o gpurun_out/full_${tag}_$k python scripts/prof_step.py 512 bf16 2 > gpurun_out/full_${tag}_$k.log 2>&1
  python scripts/ncu_summarize.py gpurun_out/full_${tag}_$k.ncu-rep "${tag} $k (cd3d 512^3, bf16 inner)" > gpurun_out/ncu_${tag}_$k.md 2>&1
  sz=$(stat -c %s gpurun_out/full_${tag}_$k.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 18000000 ]; then rm -f gpurun_out/full_${tag}_$k.ncu-rep; fi
done
timeout 600 python scripts/exp_kernels.py 512 bf16 3 > gpurun_out/exp_default_${tag}.json 2>&1
GADI_LIB=$PWD/paper_2512_21164_b200/variants/libgadi_b200_xu3.so timeout 600 python scripts/exp_kernels.py 512 bf16 3 > gpurun_out/exp_xu3_${tag}.json 2>&1

#!/bin/bash
tag=${1:-r2k}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -p no:cacheprovider tests/test_gpu_slabs.py -q -m gpu --timeout 500 -x > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
rm -f gpurun_out/peerdiag.jsonl
for args in "4 256 1 1" "8 256 0 1"; do
  timeout -s KILL 200 python scripts/peer_diag.py $args >> gpurun_out/peerdiag.jsonl 2>> gpurun_out/peerdiag.err || echo "{\"killed\": \"$args\"}" >> gpurun_out/peerdiag.jsonl
  GADI_FUSED_HALO=0 timeout -s KILL 200 python scripts/peer_diag.py $args >> gpurun_out/peerdiag.jsonl 2>> gpurun_out/peerdiag.err || echo "{\"killed\": \"$args\"}" >> gpurun_out/peerdiag.jsonl
done

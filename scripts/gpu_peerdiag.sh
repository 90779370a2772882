#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
rm -f gpurun_out/peerdiag.jsonl gpurun_out/peerdiag.err
for args in "8 64 0 1" "4 64 1 1" "8 256 0 1" "4 256 1 1"; do
  timeout -s KILL 200 python scripts/peer_diag.py $args >> gpurun_out/peerdiag.jsonl 2>> gpurun_out/peerdiag.err || echo "{\"killed\": \"$args\"}" >> gpurun_out/peerdiag.jsonl
done

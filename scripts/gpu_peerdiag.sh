#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for args in "2 64 1 1" "8 64 1 1" "8 64 0 1" "8 64 1 0" "4 256 1 1" "8 256 0 1" "8 256 1 1"; do
  timeout -s KILL 300 python scripts/peer_diag.py $args >> gpurun_out/peerdiag.jsonl 2>> gpurun_out/peerdiag.err || echo "{\"killed\": \"$args\"}" >> gpurun_out/peerdiag.jsonl
done

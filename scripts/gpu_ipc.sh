#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 scripts/ipc_check.py 16 > gpurun_out/ipc_check.log 2>&1
echo "rc=$?" >> gpurun_out/ipc_check.log

#!/bin/bash
# tools/e2e_probe.py at 1 and 4 GPUs (gpurun --gpus 4). Usage: tools/e2e_run.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/e2e_probe.py > gpurun_out/${TAG}_e2e_1.log 2>&1; echo "1 rc=$?"; grep "^n=\|copy dur" gpurun_out/${TAG}_e2e_1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/e2e_probe.py > gpurun_out/${TAG}_e2e_4.log 2>&1; echo "4 rc=$?"; grep "^n=\|copy dur" gpurun_out/${TAG}_e2e_4.log

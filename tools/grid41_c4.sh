#!/bin/bash
# The 8-GPU grid's R = 4 longitude split at full C4 scale on a 4-GPU box (JIGSAW_GRID=4x1):
# sharded-vs-single parity and the captured bench step. Usage (gpurun --gpus 4): tools/grid41_c4.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_jigsaw_gpu.py -q -s -k "c4_scale" > gpurun_out/${TAG}_c4scale.log 2>&1; echo "c4scale rc=$?"; grep "MPC4\|{'n'\|passed\|failed" gpurun_out/${TAG}_c4scale.log | tail -5
JIGSAW_GRID=4x1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 4 > gpurun_out/${TAG}_b4x1.log 2>&1; echo "bench 4x1 rc=$?"
grep '^{' gpurun_out/${TAG}_b4x1.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['parallelism'], d['clocks'])"

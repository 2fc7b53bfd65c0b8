#!/bin/bash
# Exchange ablations of the captured 2x2 C4 step (tools/overhead_probe.py; timing only).
set -u
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29751 tools/overhead_probe.py ${VARIANTS:-base nobarrier nomoments noepilogue nocomm base} > gpurun_out/${TAG}_ablate.log 2>&1; echo "rc=$?"
grep "ms/step" gpurun_out/${TAG}_ablate.log

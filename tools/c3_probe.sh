#!/bin/bash
# C3 (B = 8) at 2 GPUs: per-call breakdown of one eager step, and the captured step with one
# class of exchange operations removed at a time (timing-only ablations). gpurun --gpus 2.
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CFG=C3 B=8 timeout 600 $TR --master-port 29811 tools/phase_profile.py > gpurun_out/${TAG}_phase.log 2>&1; echo "phase rc=$?"
grep -v "^\[" gpurun_out/${TAG}_phase.log | head -30
CFG=C3 B=8 timeout 900 $TR --master-port 29812 tools/overhead_probe.py > gpurun_out/${TAG}_ablate.log 2>&1; echo "ablate rc=$?"
grep "ms/step" gpurun_out/${TAG}_ablate.log

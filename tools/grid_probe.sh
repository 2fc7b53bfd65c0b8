#!/bin/bash
# C4 (B = 1) at 4 GPUs (2x2) and C3 (B = 8) at 2 GPUs: per-call breakdown and exchange ablations.
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CFG=C4 B=1 timeout 900 $TR --nproc-per-node 4 --master-port 29821 tools/phase_profile.py > gpurun_out/${TAG}_c4_phase.log 2>&1; echo "c4 phase rc=$?"
grep -v "^\[\|Warning\|warn\|^\*\|OMP\|^$" gpurun_out/${TAG}_c4_phase.log | head -20
CFG=C4 B=1 timeout 900 $TR --nproc-per-node 4 --master-port 29822 tools/overhead_probe.py > gpurun_out/${TAG}_c4_ablate.log 2>&1; echo "c4 ablate rc=$?"
grep "ms/step" gpurun_out/${TAG}_c4_ablate.log
CFG=C3 B=8 timeout 600 $TR --nproc-per-node 2 --master-port 29823 tools/phase_profile.py > gpurun_out/${TAG}_c3_phase.log 2>&1; echo "c3 phase rc=$?"
grep -v "^\[\|Warning\|warn\|^\*\|OMP\|^$" gpurun_out/${TAG}_c3_phase.log | head -20
CFG=C3 B=8 timeout 900 $TR --nproc-per-node 2 --master-port 29824 tools/overhead_probe.py > gpurun_out/${TAG}_c3_ablate.log 2>&1; echo "c3 ablate rc=$?"
grep "ms/step" gpurun_out/${TAG}_c3_ablate.log

#!/bin/bash
# Round-end validation on a 2-GPU box after the fused-sums change: GPU test suite, smoke,
# bench at 1 (with CPU baseline) / 2 GPUs, reference arm, then the ncu launch list + GEMM
# full capture for profiles/r1h_*.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r1h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r1h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r1h_b1.log 2>&1; echo "bench1 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29912 bench.py --gpus 2 > gpurun_out/r1h_b2.log 2>&1; echo "bench2 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1h_ref.log 2>&1; echo "ref rc=$?"
for f in r1h_b1 r1h_b2 r1h_ref; do tail -1 gpurun_out/$f.log | cut -c1-600; done
timeout 900 bash tools/profile.sh r1h

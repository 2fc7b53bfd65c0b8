#!/bin/bash
# Plane-minor tile order for reduce-scatter GEMMs: probe + A/B bench at 2 and 4 GPUs + parity tests.
set -u
mkdir -p gpurun_out
for pm in 0 1; do
  if [ $pm = 1 ]; then export JG_PLANE_MAJOR=1; else unset JG_PLANE_MAJOR; fi
  echo "JG_PLANE_MAJOR=$pm"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 2959$pm tools/gemm_shape_probe.py 2>&1 | grep -E "TF/s|Error" | head -8
done
unset JG_PLANE_MAJOR
bash tools/ab.sh env:JG_PLANE_MAJOR=1 env:JG_PLANE_MINOR_DEFAULT=1 4 2
bash tools/ab.sh env:JG_PLANE_MAJOR=1 env:JG_PLANE_MINOR_DEFAULT=1 2 1
timeout 900 python -m pytest tests/test_jigsaw_gpu.py -q -x > gpurun_out/pt_pm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_pm.log

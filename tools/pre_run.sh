#!/bin/bash
# A/B: GELU pre-activations stored fp32 (A) vs operand dtype bf16 (B); parity tests for B.
set -u
mkdir -p gpurun_out
bash tools/ab.sh env:JIGSAW_PRE_FP32=1 env:JIGSAW_PRE_FP32=0 1 3
bash tools/ab.sh env:JIGSAW_PRE_FP32=1 env:JIGSAW_PRE_FP32=0 4 2
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_train_gpu.py tests/test_jigsaw_gpu.py -q -x -k "not many_blocks" > gpurun_out/pt_pre.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_pre.log

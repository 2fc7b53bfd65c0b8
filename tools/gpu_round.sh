#!/bin/bash
# One GPU validation pass of the committed tree (run under gpurun): GPU test suite (with -s so
# the parity tests' worst errors are logged), smoke, 1-GPU bench (with the CPU baseline), the
# reference arm, GEMM-vs-cuBLAS table. Usage: tools/gpu_round.sh <tag> [extra pytest args]
set -u
TAG=$1; shift
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/${TAG}_gpus.txt 2>&1; nproc >> gpurun_out/${TAG}_gpus.txt
timeout 2400 python -m pytest tests -m gpu -q -s -rs "$@" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_b1.log 2>&1; echo "bench1 rc=$?"; tail -c 600 gpurun_out/${TAG}_b1.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref1.log 2>&1; echo "ref1 rc=$?"; tail -c 400 gpurun_out/${TAG}_ref1.log
timeout 600 python tools/bench_gemm.py --json gpurun_out/${TAG}_gemm_vs_cublas.json > gpurun_out/${TAG}_gemm_vs_cublas.log 2>&1; echo "gemm rc=$?"

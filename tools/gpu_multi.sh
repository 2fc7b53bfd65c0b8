#!/bin/bash
# Multi-GPU validation on one box (run under gpurun --gpus N): Jigsaw GPU tests, C4 bench at
# 2 / N GPUs on the default grids and on the R x 1 override grids (q = R / C > 1 sub-chunks),
# the reference arm under torchrun. Usage: tools/gpu_multi.sh <tag> <N>
set -u
TAG=$1; N=$2
mkdir -p gpurun_out
run_bench () {  # <n> <logname> [env...]
  local n=$1 log=$2; shift 2
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n > gpurun_out/${TAG}_$log.log 2>&1
  echo "bench $log rc=$?"; grep '^{' gpurun_out/${TAG}_$log.log | tail -1 | cut -c1-400
}
timeout 2400 python -m pytest tests/test_jigsaw_gpu.py tests/test_cli_gpu.py -q -s -rs > gpurun_out/${TAG}_pytest_multi.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_multi.log
run_bench 2 b2
run_bench 2 b2_2x1 JIGSAW_GRID=2x1
if [ "$N" -ge 4 ]; then
  run_bench 4 b4
  run_bench 4 b4_4x1 JIGSAW_GRID=4x1
fi
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29960 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/${TAG}_ref2.log 2>&1
echo "ref2 rc=$?"; grep -c '^{' gpurun_out/${TAG}_ref2.log

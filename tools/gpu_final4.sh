#!/bin/bash
# Round-close multi-GPU check (gpurun --gpus 4): C4 bench at 2 and 4 GPUs (default grids) and the
# R x 1 grids, the reference arm under torchrun. Usage: tools/gpu_final4.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run () { local n=$1 log=$2; shift 2
  env "$@" timeout 900 $TR --nproc-per-node $n --master-port $((29900 + n + ${#log})) bench.py --gpus $n > gpurun_out/${TAG}_$log.log 2>&1
  echo "$log rc=$?"; grep '^{' gpurun_out/${TAG}_$log.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d.get('comm') or {}
print(' ', d['n_gpus'], round(d['value'],2), 'samples/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], 'MHz, e2e', round(d['e2e']['value'],2), 'gemm frac', round(d['roofline']['frac'],3), 'comm', c.get('grid'), c.get('nvlink_bytes_per_step_per_rank'), round(c.get('frac', 0), 3))"; }
run 2 b2 X=1
run 4 b4 X=1
run 2 b2_2x1 JIGSAW_GRID=2x1
run 4 b4_4x1 JIGSAW_GRID=4x1
timeout 900 $TR --nproc-per-node 2 --master-port 29990 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/${TAG}_ref2.log 2>&1
echo "ref2 rc=$?"; grep -c '^{' gpurun_out/${TAG}_ref2.log

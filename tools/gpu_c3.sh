#!/bin/bash
# C3 strong scaling (B = 8) at 1 / 2 / 4 GPUs, host->device feed probe, Jigsaw GPU tests.
# Usage (gpurun --gpus 4): tools/gpu_c3.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_jigsaw_gpu.py -q -s -rs ${PYTEST_K:-} > gpurun_out/${TAG}_pytest_multi.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_multi.log
timeout 600 python bench.py --config C3 --batch 8 --no-cpu-baseline > gpurun_out/${TAG}_c3_1.log 2>&1; echo "c3 n1 rc=$?"
for n in 2 4; do timeout 600 $TR --nproc-per-node $n --master-port $((29700 + n)) bench.py --gpus $n --config C3 --batch 8 > gpurun_out/${TAG}_c3_$n.log 2>&1; echo "c3 n$n rc=$?"; done
for n in 1 2 4; do grep '^{' gpurun_out/${TAG}_c3_$n.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['n_gpus'], round(d['value'],1), 'samples/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'])"; done
timeout 300 $TR --nproc-per-node 4 --master-port 29790 tools/h2d_probe.py > gpurun_out/${TAG}_h2d.log 2>&1; echo "h2d rc=$?"; grep H2D gpurun_out/${TAG}_h2d.log

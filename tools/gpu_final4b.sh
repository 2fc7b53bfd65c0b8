#!/bin/bash
# Round-close multi-GPU pass (gpurun --gpus 4): every multi-GPU test, C4 at 2 / 4 GPUs,
# C3 (B = 8) at 1 / 2 / 4, C5 weak scaling at 2 / 4. Usage: tools/gpu_final4b.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_jigsaw_gpu.py tests/test_cli_gpu.py -q -s -rs > gpurun_out/${TAG}_pytest_multi.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_multi.log
line () { grep '^{' $1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d.get('comm') or {}
print(' ', d['config']['workload'][:3], d['n_gpus'], round(d['value'],2), 'samples/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], 'MHz e2e', round(d['e2e']['value'],2), 'tflops', round(d['tflops'],1))"; }
for n in 2 4; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29600 + n)) bench.py --gpus $n > gpurun_out/${TAG}_c4_$n.log 2>&1; echo "c4 n$n rc=$?"; line gpurun_out/${TAG}_c4_$n.log
done
timeout 600 python bench.py --config C3 --batch 8 --no-cpu-baseline > gpurun_out/${TAG}_c3_1.log 2>&1; echo "c3 n1 rc=$?"; line gpurun_out/${TAG}_c3_1.log
for n in 2 4; do
  timeout 600 $TR --nproc-per-node $n --master-port $((29610 + n)) bench.py --gpus $n --config C3 --batch 8 > gpurun_out/${TAG}_c3_$n.log 2>&1; echo "c3 n$n rc=$?"; line gpurun_out/${TAG}_c3_$n.log
done
for n in 2 4; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29620 + n)) bench.py --gpus $n --config C5 > gpurun_out/${TAG}_c5_$n.log 2>&1; echo "c5 n$n rc=$?"; line gpurun_out/${TAG}_c5_$n.log
done

#!/bin/bash
# Final check of the round's tree on one 4-GPU box: the whole GPU suite, smoke, C4 bench at
# 1 / 2 / 4 GPUs. Usage (gpurun --gpus 4): tools/gpu_close.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
line () { grep '^{' $1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(' ', d['n_gpus'], round(d['value'],2), 'samples/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], 'MHz e2e', round(d['e2e']['value'],2), 'gemm frac', round(d['roofline']['frac'],3))"; }
timeout 900 python bench.py > gpurun_out/${TAG}_b1.log 2>&1; echo "b1 rc=$?"; line gpurun_out/${TAG}_b1.log
for n in 2 4; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29700 + n)) bench.py --gpus $n > gpurun_out/${TAG}_b$n.log 2>&1; echo "b$n rc=$?"; line gpurun_out/${TAG}_b$n.log
done

#!/bin/bash
# Round-end check of the driver's own commands on one 4-GPU box: `python bench.py` (defaults,
# CPU baseline included), the reference arm, torchrun C4 at 2 / 4 GPUs (+ reference arm at 4),
# C3 at 1 / 2 / 4. Usage (gpurun --gpus 4): tools/gpu_round_end.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
line () { grep '^{' $1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d.get('clocks') or {}; e=d.get('e2e') or {}
print(' ', d.get('impl', 'ours'), d['n_gpus'], d['config'].get('workload', '')[:3], round(d['value'], 4), d['unit'], round(d['ms_per_step'], 2), 'ms', c.get('sm_mhz'), 'MHz', c.get('reasons'), 'e2e', e.get('value') and round(e['value'], 3), 'frac', (d.get('roofline') or {}).get('frac'))"; }
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/${TAG}_b1.log 2>&1; echo "bench default rc=$? $(( $(date +%s) - t0 )) s"; line gpurun_out/${TAG}_b1.log
t0=$(date +%s); timeout 1200 python bench.py --impl reference > gpurun_out/${TAG}_ref1.log 2>&1; echo "ref default rc=$? $(( $(date +%s) - t0 )) s"; line gpurun_out/${TAG}_ref1.log
for n in 2 4; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29800 + n)) bench.py --gpus $n > gpurun_out/${TAG}_b$n.log 2>&1; echo "b$n rc=$?"; line gpurun_out/${TAG}_b$n.log
done
t0=$(date +%s); timeout 1200 $TR --nproc-per-node 4 --master-port 29810 bench.py --impl reference --gpus 4 > gpurun_out/${TAG}_ref4.log 2>&1; echo "ref4 rc=$? $(( $(date +%s) - t0 )) s"; grep -c '^{' gpurun_out/${TAG}_ref4.log; line gpurun_out/${TAG}_ref4.log
timeout 600 python bench.py --config C3 --batch 8 --no-cpu-baseline > gpurun_out/${TAG}_c3_1.log 2>&1; echo "c3 1 rc=$?"; line gpurun_out/${TAG}_c3_1.log
for n in 2 4; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29820 + n)) bench.py --gpus $n --config C3 --batch 8 > gpurun_out/${TAG}_c3_$n.log 2>&1; echo "c3 $n rc=$?"; line gpurun_out/${TAG}_c3_$n.log
done

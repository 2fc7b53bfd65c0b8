set -u
python -m pytest tests/test_guards_gpu.py -q -x > gpurun_out/r2q_guards.log 2>&1; echo guards rc=$?; tail -1 gpurun_out/r2q_guards.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29931 bench.py --gpus 4 > gpurun_out/r2q_b4.log 2>&1; echo b4 rc=$?
grep '^{' gpurun_out/r2q_b4.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],2), round(d['e2e']['device_ms_per_call'],2))"
timeout 900 python -m pytest tests/test_jigsaw_gpu.py -q -x -k "nccl_parity or override or captured" > gpurun_out/r2q_multi.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/r2q_multi.log

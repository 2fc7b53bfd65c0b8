#!/bin/bash
# Validation + bench on a 4-GPU box: Jigsaw GPU tests, then bench at 1 / 2 / 4 GPUs.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jigsaw_gpu.py tests/test_train_gpu.py -q > gpurun_out/pytest_val.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_val.log
timeout 300 python bench.py > gpurun_out/bv1.log 2>&1
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2970$n bench.py --gpus $n > gpurun_out/bv$n.log 2>&1
done
for n in 1 2 4; do
python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bv{n}.log").read().strip().splitlines()[-1])
    print(n, round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2), d["clocks"]["sm_mhz"])
except Exception as e:  # noqa: BLE001
    print(n, "FAILED", e)
PY
done

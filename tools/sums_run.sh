#!/bin/bash
# Validation of the fused bias-gradient sums in the LN backward pass: full GPU suite + benches.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_sums.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sums.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s1.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29934 bench.py --gpus 4 > gpurun_out/s4.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29932 bench.py --gpus 2 > gpurun_out/s2.log 2>&1
for f in s1 s2 s4; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{f}.log").read().strip().splitlines()[-1])
    print(f, round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2), d["clocks"]["sm_mhz"])
except Exception as e:  # noqa: BLE001
    print(f, "FAILED", e)
PY
done

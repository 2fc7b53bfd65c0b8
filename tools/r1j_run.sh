#!/bin/bash
# Final round-1 check of the committed tree on a 4-GPU box: GPU suite, smoke, bench 1 (with the
# CPU baseline) / 2 / 4 GPUs, reference arm at N = 1 and under torchrun N = 2.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r1j.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r1j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r1j_b1.log 2>&1; echo "bench1 rc=$?"
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2995$n bench.py --gpus $n > gpurun_out/r1j_b$n.log 2>&1; echo "bench$n rc=$?"
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29960 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/r1j_ref2.log 2>&1; echo "ref2 rc=$?"
grep -c '^{' gpurun_out/r1j_ref2.log
for n in 1 2 4; do
python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r1j_b{n}.log").read().strip().splitlines()[-1])
    print(n, round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2), d["clocks"]["sm_mhz"],
          "gemm_frac", round(d["roofline"]["frac"], 3), "cpu", d.get("cpu_baseline", {}).get("value"))
except Exception as e:  # noqa: BLE001
    print(n, "FAILED", e)
PY
done

#!/bin/bash
# Round-end validation on a 4-GPU box: full GPU test suite (n = 2, 4 Jigsaw + DP replicas), smoke,
# bench at 1 / 2 / 4 GPUs, CLI dp (C2, mp 2 x 1/2 replicas) and weak (C5 at 2 / 4) suites.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r1i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r1i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r1i_b1.log 2>&1; echo "bench1 rc=$?"
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2993$n bench.py --gpus $n > gpurun_out/r1i_b$n.log 2>&1; echo "bench$n rc=$?"
done
timeout 600 python -m paper_2507_05753_b200 bench dp --mp 2 --workload C2 --steps 5 --warmup 3 --out gpurun_out/r1i_suites > gpurun_out/r1i_dp.log 2>&1; echo "dp rc=$?"
timeout 900 python -m paper_2507_05753_b200 bench weak --steps 3 --warmup 3 --out gpurun_out/r1i_suites > gpurun_out/r1i_weak.log 2>&1; echo "weak rc=$?"
python -m paper_2507_05753_b200 report gpurun_out/r1i_suites/*.csv 2>&1
for n in 1 2 4; do
python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r1i_b{n}.log").read().strip().splitlines()[-1])
    print(n, round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2), d["clocks"]["sm_mhz"])
except Exception as e:  # noqa: BLE001
    print(n, "FAILED", e)
PY
done

#!/bin/bash
# Round-1 validation + A/B: full GPU test suite, smoke, then bench at 2 and 4 GPUs with the
# jg_group_barrier (default) and torch symmetric-memory barriers.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for n in 2 4; do for b in jg torch; do
  JIGSAW_BARRIER=$b timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 296$n${#b} bench.py --gpus $n > gpurun_out/b${n}_$b.log 2>&1
  python - "$n" "$b" <<'PY'
import json, sys
n, b = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/b{n}_{b}.log").read().strip().splitlines()[-1])
    print(n, b, round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2))
except Exception as e:  # noqa: BLE001
    print(n, b, "FAILED", e)
PY
done; done

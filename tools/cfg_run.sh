#!/bin/bash
# Other BASELINE configs on one 4-GPU box (C3 strong scaling at 1 / 2 / 4 with B = 8; C5 weak scaling: run C5 2; run C5 4).
set -u
mkdir -p gpurun_out
run() {  # config n [bench args]
  c=$1; n=$2; shift 2
  if [ "$n" = 1 ]; then timeout 400 python bench.py --config $c --no-cpu-baseline "$@" > gpurun_out/cfg_${c}_$n.log 2>&1
  else timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 298$n$((RANDOM % 9)) bench.py --gpus $n --config $c "$@" > gpurun_out/cfg_${c}_$n.log 2>&1; fi
  python - "$c" "$n" <<'PY'
import json, sys
c, n = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/cfg_{c}_{n}.log").read().strip().splitlines()[-1])
    print(c, n, d["scaling"], round(d["value"], 3), "samples/s", round(d["ms_per_step"], 3), "ms", round(d["tflops"], 1),
          "TFLOP/s", d["config"]["params"], "params", "gemm", round(d["roofline"]["achieved"], 1), d["clocks"]["sm_mhz"])
except Exception as e:  # noqa: BLE001
    print(c, n, "FAILED", e, open(f"gpurun_out/cfg_{c}_{n}.log").read()[-1500:])
PY
}
run C3 1 --batch 8; run C3 2 --batch 8; run C3 4 --batch 8

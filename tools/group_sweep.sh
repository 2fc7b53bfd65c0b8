#!/bin/bash
# A/B of the GEMM L2 tile-group height (JG_TILE_GROUP_M) on 1 GPU: prebuilt variants in
# tools/variants/g<G>.so swapped in before each bench run (8 = the default, run first and last).
set -u
mkdir -p gpurun_out
for G in 8 4 16 32 8; do
  cp tools/variants/g$G.so paper_2507_05753_b200/libjigsaw_sm100.so
  timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/gs_$G.log 2>&1
  python - "$G" <<'PY'
import json, sys
G = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/gs_{G}.log").read().strip().splitlines()[-1])
    print("G", G, round(d["value"], 3), "ms", round(d["ms_per_step"], 3), "gemm_frac", round(d["roofline"]["frac"], 4),
          "sm_mhz", d["clocks"]["sm_mhz"])
except Exception as e:  # noqa: BLE001
    print("G", G, "FAILED", e)
PY
done

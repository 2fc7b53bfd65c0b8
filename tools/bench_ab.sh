#!/bin/bash
# 1-GPU bench A/B of library variants (tools/variants/<name>.so via JIGSAW_LIB; "base" = in-tree),
# interleaved over rounds: samples/s, ms, SM clock median, J per step (NVML).
# Usage: tools/bench_ab.sh <tag> <rounds> base v1 [v2 ...]
set -u
TAG=$1; ROUNDS=$2; shift 2
mkdir -p gpurun_out
for round in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2507_05753_b200/libjigsaw_sm100.so; else lib=tools/variants/$v.so; fi
    JIGSAW_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_${v}_r$round.log 2>&1
    grep '^{' gpurun_out/${TAG}_${v}_r$round.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']
print('$v', round(d['value'],2), round(d['ms_per_step'],2), c['sm_mhz'], c.get('energy_j_per_step'), c.get('avg_power_w'), 'gemm frac', round(d['roofline']['frac'],3))"
  done
done

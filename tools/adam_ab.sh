#!/bin/bash
# A/B of streaming cache hints in the Adam kernel (JG_ADAM_CS) on 1 GPU: HBM micro-bench + bench.
set -u
mkdir -p gpurun_out
for V in base cs base cs; do
  cp tools/variants/$V.so paper_2507_05753_b200/libjigsaw_sm100.so
  echo "== $V"; timeout 120 python tools/membench.py --only adam 2>&1 | grep "| adam"
done
for V in base cs base cs; do
  cp tools/variants/$V.so paper_2507_05753_b200/libjigsaw_sm100.so
  timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/aab_$V.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/aab_$V.log').read().strip().splitlines()[-1]);print('$V',round(d['value'],3),round(d['ms_per_step'],3),d['clocks']['sm_mhz'])"
done

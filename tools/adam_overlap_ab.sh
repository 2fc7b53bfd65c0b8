#!/bin/bash
# Adam overlapped with the backward (side stream, SM-pinned) vs after it: parity tests, then
# alternating bench lines. Usage: tools/adam_overlap_ab.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_train_gpu.py tests/test_bench_parity_gpu.py -q -s -x -k "not full_depth" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log; grep "C3 \|C4 " gpurun_out/${TAG}_pytest.log | head -4
for round in 1 2; do
  for v in "0 16" "1 16" "1 24" "1 8"; do
    set -- $v
    JIGSAW_ADAM_OVERLAP=$1 JIGSAW_ADAM_SMS=$2 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_o$1_s$2_r$round.log 2>&1
    grep '^{' gpurun_out/${TAG}_o$1_s$2_r$round.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('overlap=$1 sms=$2', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
  done
done

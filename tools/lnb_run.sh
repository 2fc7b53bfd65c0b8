#!/bin/bash
# A/B of the layer-norm backward with fused row sums (1 GPU): kernel tests, HBM micro-bench, bench.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x > gpurun_out/lnb_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/lnb_pytest.log
timeout 300 python tools/membench.py --only ln_bwd > gpurun_out/lnb_membench.log 2>&1; echo "membench rc=$?"; grep -v "^{" gpurun_out/lnb_membench.log | tail -8
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/lnb_b1.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/lnb_b1.log').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['clocks'])"

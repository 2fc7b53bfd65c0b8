#!/bin/bash
# Round-close validation on 1 GPU: GPU test suite, smoke, the bench line (with the CPU baseline),
# the reference arm, fused-Adam and f32-mode bench lines, ncu launch list + GEMM full capture of
# the bench command (summaries into gpurun_out/profiles). Usage: tools/gpu_final1.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out/profiles
timeout 2400 python -m pytest tests -m gpu -q -s -rs > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_b1.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref1.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --no-cpu-baseline --fused-adam > gpurun_out/${TAG}_b1_fusedadam.log 2>&1; echo "fused-adam rc=$?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_b1_again.log 2>&1; echo "bench again rc=$?"
timeout 600 python bench.py --no-cpu-baseline --config C2 --batch 32 --dtype f32 > gpurun_out/${TAG}_c2_f32.log 2>&1; echo "c2 f32 rc=$?"
timeout 600 python bench.py --no-cpu-baseline --config C2 --batch 32 > gpurun_out/${TAG}_c2_bf16.log 2>&1; echo "c2 bf16 rc=$?"
for f in b1 b1_fusedadam b1_again c2_f32 c2_bf16; do grep '^{' gpurun_out/${TAG}_$f.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'gemm frac', round(d['roofline']['frac'],3))" 2>/dev/null; done
bash tools/profile.sh $TAG > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"
NCU_SUMMARY_OUT=gpurun_out/profiles python tools/ncu_summary.py $TAG --launches gpurun_out/launches_$TAG.csv \
  --full gpurun_out/prof_gemm_$TAG.ncu-rep > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/prof_gemm_$TAG.ncu-rep
ls gpurun_out/profiles

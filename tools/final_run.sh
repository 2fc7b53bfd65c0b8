#!/bin/bash
# End-of-round validation on a 4-GPU box: full GPU test suite, smoke, bench at 1 (with the CPU
# baseline) / 2 / 4 GPUs.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final1.log 2>&1
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2990$n bench.py --gpus $n > gpurun_out/final$n.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.log 2>&1
for f in final1 final2 final4 final_ref; do tail -1 gpurun_out/$f.log | cut -c1-400; done

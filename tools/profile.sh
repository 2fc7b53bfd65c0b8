#!/bin/bash
# ncu evidence for the bench command (run under gpurun; 1 GPU). Usage: tools/profile.sh <tag> [bench args]
set -u
TAG=$1; shift
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --no-graph $*"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_$TAG.log 2>&1
echo launches rc=$?
python bench.py $ARGS > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 3 \
    -o gpurun_out/prof_gemm_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc=$?

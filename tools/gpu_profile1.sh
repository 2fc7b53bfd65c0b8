#!/bin/bash
# ncu launch list + GEMM full capture of the 1-GPU bench command, summarised into
# gpurun_out/profiles (tools/profile.sh, tools/ncu_summary.py). Usage: tools/gpu_profile1.sh <tag>
set -u
TAG=$1
mkdir -p gpurun_out/profiles
bash tools/profile.sh $TAG > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"; cat gpurun_out/${TAG}_profile.log
NCU_SUMMARY_OUT=gpurun_out/profiles python tools/ncu_summary.py $TAG --launches gpurun_out/launches_$TAG.csv \
  --full gpurun_out/prof_gemm_$TAG.ncu-rep > gpurun_out/${TAG}_summary.log 2>&1; echo "summary rc=$?"
rm -f gpurun_out/prof_gemm_$TAG.ncu-rep
ls gpurun_out/profiles

#!/bin/bash
# A/B of GEMM library variants (tools/variants/*.so via JIGSAW_LIB) on the operand-major probe,
# alternating variants over two rounds. Usage: tools/ab_gemm_variants.sh <tag> base v1 [v2 ...]
set -u
TAG=$1; shift
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="tools/variants/$v.so"; fi
    echo "== $v round $round"
    JIGSAW_LIB=${lib:-paper_2507_05753_b200/libjigsaw_sm100.so} timeout 300 python tools/gemm_majors.py 2>&1 | tail -4
  done
done > gpurun_out/${TAG}_ab.log 2>&1
cat gpurun_out/${TAG}_ab.log

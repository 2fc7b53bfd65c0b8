#!/bin/bash
# HBM-kernel A/B: the in-tree library against variants (tools/variants/<name>.so), 2x2 tiles.
# Usage: tools/hbm_ab.sh <tag> <variant> [<variant> ...]
set -u
TAG=$1; shift
for round in 1 2; do
  echo "== base $round"; python tools/membench.py --tile 2x2 --reps 30 2>&1 | grep -E "^\| (epilogue|ln_apply|patchify|colsum)"
  for V in "$@"; do
    echo "== $V $round"; JIGSAW_LIB=tools/variants/$V.so python tools/membench.py --tile 2x2 --reps 30 2>&1 | grep -E "^\| (epilogue|ln_apply|patchify|colsum)"
  done
done > gpurun_out/${TAG}_hbm_ab.log 2>&1
cat gpurun_out/${TAG}_hbm_ab.log

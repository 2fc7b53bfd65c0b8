#!/bin/bash
# compute-sanitizer over the small-shape kernel workload (one tool per gpurun call):
#   tools/sanitize.sh <tag> memcheck|racecheck|synccheck|initcheck
set -u
TAG=$1; TOOL=$2
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool $TOOL --print-limit 50 --target-processes all \
  python tools/sanitize_cases.py > gpurun_out/${TAG}_sanitize_${TOOL}.log 2>&1
echo "$TOOL rc=$?"; tail -4 gpurun_out/${TAG}_sanitize_${TOOL}.log

#!/bin/bash
# A/B timing on the same box, alternating runs so power and clock drift hit both equally.
# A / B: a build of libjigsaw_sm100.so (path) or environment settings ("env:VAR=val[,VAR2=val]").
# Usage (under gpurun): tools/ab.sh <A> <B> <n_gpus> [rounds] [bench args]
set -u
A=$1; B=$2; N=$3; ROUNDS=${4:-3}; shift 4 2>/dev/null || shift $#
mkdir -p gpurun_out
for r in $(seq 1 $ROUNDS); do
  for tag in A B; do
    spec=$A; [ $tag = B ] && spec=$B
    if [[ $spec == env:* ]]; then
      ENVS=$(echo ${spec#env:} | tr ',' ' ')
    else
      ENVS="JIGSAW_LIB=$spec"
    fi
    if [ "$N" = 1 ]; then
      env $ENVS timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.json 2>/dev/null
    else
      env $ENVS timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 \
        --master-port $((29600 + r)) --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline "$@" \
        > gpurun_out/ab_$tag.json 2>/dev/null
    fi
    python - "$tag" "$r" <<'PY'
import json, sys
tag, r = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ab_{tag}.json").read().strip().splitlines()[-1])
print(f"round {r} {tag}: {d['value']:.2f} samples/s  {d['ms_per_step']:.3f} ms  sm {d['clocks']['sm_mhz']} MHz")
PY
  done
done

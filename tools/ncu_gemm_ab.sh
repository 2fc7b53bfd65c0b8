#!/bin/bash
# Clock-locked (ncu --clock-control base) GEMM time of one eager C4 step per library build:
# isolates kernel efficiency from the power-cap clock swings that dominate wall-time A/B.
# Usage (under gpurun): tools/ncu_gemm_ab.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  JIGSAW_LIB=$lib timeout 600 ncu --clock-control base -k regex:gemm_kernel --launch-skip 41 --launch-count 41 \
    --metrics gpu__time_duration.sum --csv python tools/ncu_step.py --steps 2 > gpurun_out/ncuab_$tag.csv 2>/dev/null
  python - "$tag" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ncuab_{tag}.csv")) if len(r) > 10]
hdr = rows[0]; i = hdr.index("Metric Value"); u = hdr.index("Metric Unit")
vals = [float(r[i].replace(",", "")) * (1e-3 if r[u] == "nsecond" else 1.0) for r in rows[1:]]
print(f"{tag}: {len(vals)} GEMMs {sum(vals)/1e3:.3f} ms (base clock)  per-launch us: {' '.join(f'{v:.0f}' for v in vals[:20])}")
PY
done

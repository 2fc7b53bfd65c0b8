#!/bin/bash
# ncu --set full of single jg_gemm shapes (run under gpurun, 1 GPU): TN vs NT at C4 sizes.
set -u
TAG=$1
mkdir -p gpurun_out
for spec in "4320 8640 16380 1 1" "16380 4320 8640 0 0" "4480 4320 16380 1 1" "16380 8640 4320 0 1"; do
  name=$(echo $spec | tr ' ' '_')
  python tools/gemm_probe.py $spec > gpurun_out/${TAG}_probe_$name.log 2>&1 || { echo "probe $name failed"; continue; }
  cat gpurun_out/${TAG}_probe_$name.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_gemm_$name python tools/gemm_probe.py $spec 4 > gpurun_out/${TAG}_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  rep=gpurun_out/${TAG}_gemm_$name.ncu-rep
  ncu -i $rep --page raw --csv > gpurun_out/${TAG}_gemm_${name}_raw.csv 2>/dev/null
  ncu -i $rep --page details --csv > gpurun_out/${TAG}_gemm_${name}_details.csv 2>/dev/null
  ncu -i $rep --page source --csv > gpurun_out/${TAG}_gemm_${name}_source.csv 2>/dev/null
  gzip -f gpurun_out/${TAG}_gemm_${name}_source.csv
  rm -f $rep  # reports are large: keep the csv exports (gpurun copies back <= 64 MiB)
done

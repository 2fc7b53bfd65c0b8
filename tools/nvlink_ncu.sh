#!/bin/bash
# NVLink counters of the peer-store GEMM (gpurun --gpus 2; one process drives both GPUs).
set -u
TAG=$1
mkdir -p gpurun_out
python tools/nvlink_probe.py > gpurun_out/${TAG}_nvlink_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/${TAG}_nvlink_probe.log
ncu --query-metrics > gpurun_out/${TAG}_ncu_metrics.txt 2>&1
grep -i "nvl" gpurun_out/${TAG}_ncu_metrics.txt | head -40 > gpurun_out/${TAG}_ncu_nvl_metrics.txt
cat gpurun_out/${TAG}_ncu_nvl_metrics.txt | head -40
M=$(grep -io "^nvl[a-z_]*__[a-z_]*" gpurun_out/${TAG}_ncu_metrics.txt | sort -u | head -12 | sed 's/$/.sum/' | paste -sd, -)
echo "metrics: $M"
if [ -n "$M" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,$M --clock-control none \
    -k regex:gemm_kernel -c 8 --csv python tools/nvlink_probe.py --reps 1 > gpurun_out/${TAG}_nvlink_ncu.csv 2>&1
  echo "ncu rc=$?"; tail -40 gpurun_out/${TAG}_nvlink_ncu.csv
fi
rm -f gpurun_out/${TAG}_ncu_metrics.txt

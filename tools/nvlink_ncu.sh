#!/bin/bash
# NVLink counters of the peer-store GEMM (gpurun --gpus 2; one process drives both GPUs).
set -u
TAG=$1
mkdir -p gpurun_out
python tools/nvlink_probe.py > gpurun_out/${TAG}_nvlink_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/${TAG}_nvlink_probe.log
ncu --query-metrics > gpurun_out/${TAG}_ncu_metrics.txt 2>&1
grep -i "nvl" gpurun_out/${TAG}_ncu_metrics.txt | head -40 > gpurun_out/${TAG}_ncu_nvl_metrics.txt
cat gpurun_out/${TAG}_ncu_nvl_metrics.txt | head -40
M=nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvltx__cycles_active.sum,nvltx__cycles_elapsed.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum
echo "metrics: $M"
if [ -n "$M" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,$M --clock-control none \
    -k regex:gemm_kernel -c 8 --csv python tools/nvlink_probe.py --reps 1 > gpurun_out/${TAG}_nvlink_ncu.csv 2>&1
  echo "ncu rc=$?"; grep -E "gpu__time|nvltx__bytes|nvltx__cycles|nvlrx__bytes.sum" gpurun_out/${TAG}_nvlink_ncu.csv | awk -F'","' '{print $1, $(NF-2), $NF}' | head -60
fi
rm -f gpurun_out/${TAG}_ncu_metrics.txt

set -u
for cap in 148 132 148 132; do
  JG_GEMM_SMS=$cap timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2u_cap$cap.log 2>&1
  grep '^{' gpurun_out/r2u_cap$cap.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cap', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'gemm', round(d['roofline']['achieved'],0))"
done

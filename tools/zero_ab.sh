set -u
for r in 1 2 3; do for v in 0 1; do
JIGSAW_TORCH_ZERO=$v timeout 600 python bench.py --no-cpu-baseline 2>&1 | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('torch_zero=$v', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done; done

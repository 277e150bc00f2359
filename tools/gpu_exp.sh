for cfg in "0 16 2" "1 16 2" "0 0 2" "0 16 2"; do
  set -- $cfg
  SOS_DEBUG_NODRAIN=$1 SOS_SKEW_EPOCH=$2 SOS_SKEW_LAG=$3 timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$cfg', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done

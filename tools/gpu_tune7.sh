for rep in 1 2; do
for cfg in "4 2 8" "8 2 8" "16 2 8" "4 3 8" "0 2 8"; do
  set -- $cfg
  SOS_SKEW_EPOCH=$1 SOS_SKEW_LAG=$2 SOS_TILE_GROUP=$3 timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$cfg', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done; done

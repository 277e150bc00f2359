# K-skew / tile-group sweep of the int8 GEMMs (bench.py, config 4)
for cfg in "16 2 8" "32 2 8" "8 2 8" "16 1 8" "16 3 8" "16 2 4" "16 2 16" "0 2 8"; do
  set -- $cfg
  SOS_SKEW_EPOCH=$1 SOS_SKEW_LAG=$2 SOS_TILE_GROUP=$3 timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$cfg', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done

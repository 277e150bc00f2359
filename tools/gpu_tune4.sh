for cfg in "4 2 8" "4 4 8" "4 8 8" "8 3 8" "4 16 8"; do
  set -- $cfg
  SOS_SKEW_EPOCH=$1 SOS_SKEW_LAG=$2 SOS_TILE_GROUP=$3 timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  SOS_GEMM_STATS=1 SOS_SKEW_EPOCH=$1 SOS_SKEW_LAG=$2 SOS_TILE_GROUP=$3 timeout 200 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "mode=2" | tail -1 > /tmp/s.txt
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$cfg', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'], '|', open('/tmp/s.txt').read().strip()[40:])"
done

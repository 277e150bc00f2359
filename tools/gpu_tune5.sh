for rep in 1 2; do
for sl in 256 64 16 0; do
  SOS_SKEW_SLEEP=$sl timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('sleep $sl', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done; done

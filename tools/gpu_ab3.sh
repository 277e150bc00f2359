cd paper_2410_19844_b200
for rep in 1; do for v in s5 s4 s5 s4; do
  cp libsos_$v.so libsos_b200.so
  (cd .. && timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null)
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$v', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done; done
cp libsos_s5.so libsos_b200.so

# A/B of two library builds on the same box (bench + ncu imma activity)
cd paper_2410_19844_b200
for rep in 1 2; do
for v in orig alt; do
  cp libsos_$v.so libsos_b200.so
  (cd .. && timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null)
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('$v', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done; done
for v in orig alt; do
  cp libsos_$v.so libsos_b200.so
  (cd .. && timeout 300 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemmq -s 3 -c 2 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_gemmq<|imma|tc_cycles|duration|per_second" | sed "s/^/$v /")
done
cp libsos_orig.so libsos_b200.so

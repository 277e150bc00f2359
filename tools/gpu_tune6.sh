timeout 300 python -m pytest tests -x -q -m gpu -k "forward_parity or backward_parity or descend_matches" > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
for rep in 1 2 3; do
  timeout 200 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('A-ordered', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"
done
timeout 300 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemmq -s 3 -c 2 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_gemmq|imma|tc_cycles|duration|per_second" > gpurun_out/tune6_ncu.txt

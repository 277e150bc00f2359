timeout 600 python -m pytest tests -x -q -m gpu -k "forward_parity or backward_parity or descend_matches or full_size or segmented" > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 300 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemmq -s 3 -c 2 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_gemmq<|imma|duration|per_second"
for i in 1 2; do timeout 300 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null; python3 -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']
print('elect+prod', round(d['value'],3), 'fwd', round(k['gemm_fwd']['ms_per_launch'],2), 'bwd', round(k['gemm_bwd']['ms_per_launch'],2), 'clk', d['clocks']['sm_mhz'])"; done

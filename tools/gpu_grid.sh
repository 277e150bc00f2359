for c in 148 112 74 38; do
  SOS_GEMM_CTAS=$c timeout 300 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemmq -s 3 -c 2 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_gemmq<|imma|duration|per_second|lts__" | sed "s/^/ctas$c /"
done

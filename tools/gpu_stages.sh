cd paper_2410_19844_b200
for v in s5 s4 s3; do
  cp libsos_$v.so libsos_b200.so
  (cd .. && timeout 300 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemmq -s 3 -c 2 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_gemmq<|imma|duration|per_second" | sed "s/^/$v /")
done
cp libsos_s5.so libsos_b200.so

# what the fused update costs inside the backward: the same descent with the fused step (update in the
# backward's epilogue warps) vs the split step (backward stores the gradient, k_update_rows applies it),
# per-kernel times and DRAM bytes from an ncu launch list
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
for shape in "12 6 12376" "17 5 20349"; do
  for sp in 0 1; do
    timeout 300 python tools/time_shape.py $shape 10 split=$sp --kernels
    timeout 600 ncu --metrics $M --clock-control none -c 40 --csv --log-file "gpurun_out/p2_upd_${shape// /_}_split$sp.csv" python tools/time_shape.py $shape 3 split=$sp > /dev/null 2>&1
  done
done 2>&1 | tee gpurun_out/p2_update_cost.log

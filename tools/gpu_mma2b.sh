nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/m2 tools/mma2_bench.cu
/tmp/m2 160 0 1.5 0; /tmp/m2 160 0 1.5 1; /tmp/m2 160 1 1.5 0; /tmp/m2 160 1 1.5 1
for p in 0 1; do timeout 120 ncu --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second -c 2 /tmp/m2 160 1 0.3 $p 2>&1 | grep -E "imma|per_second" | sed "s/^/pattern$p /"; done

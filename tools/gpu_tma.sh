nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tb tools/tma_bench.cu -lcuda
for m in 0 3 4; do /tmp/tb $m; done

nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tb tools/tma_bench.cu -lcuda
for c in 148 112 74 38 16; do echo "ctas $c"; /tmp/tb 0 $c | tail -1; done

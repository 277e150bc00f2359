nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mp tools/mma_power.cu -lcuda
for n in 64 96 128 160 192 224 256; do /tmp/mp 5 1.5 $n; done
for n in 128 160 256; do /tmp/mp 2 1.5 $n; done

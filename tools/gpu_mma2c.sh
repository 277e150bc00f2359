nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/m2 tools/mma2_bench.cu
for sw in 0 1 2 3; do /tmp/m2 160 0 1.0 1 $sw; done

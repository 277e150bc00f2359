// Cost of cooperative launches and grid barriers on this GPU (k_mid design):
// an (almost) empty cooperative kernel with S grid.sync()s, blocks x 256 threads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int syncs, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int s = 0; s < syncs; ++s) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = syncs;
}
__global__ void plain(int* out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 1;
}
int main() {
    int* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks : {48, 148, 296, 592}) {
        for (int syncs : {0, 1, 2, 4, 8}) {
            void* args[] = {&syncs, &out};
            for (int w = 0; w < 20; ++w) cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
            cudaEventRecord(a);
            for (int it = 0; it < 200; ++it) cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("coop blocks=%d syncs=%d: %.2f us per launch\n", blocks, syncs, ms * 1e3 / 200);
        }
        for (int w = 0; w < 20; ++w) plain<<<blocks, 256>>>(out);
        cudaEventRecord(a);
        for (int it = 0; it < 200; ++it) plain<<<blocks, 256>>>(out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("plain blocks=%d: %.2f us per launch\n", blocks, ms * 1e3 / 200);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}

// mma2_bench.cu -- microbenchmark: sustained tcgen05.mma.cta_group::2.kind::i8
// throughput (M = 256 over a CTA pair) versus N, operands resident in shared
// memory (SWIZZLE_64B K-major, zeros or random bytes), one accumulator per N.
// Answers: how close to the s8 peak can an N=160 pair MMA run by itself?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma2_bench tools/mma2_bench.cu
//   ./mma2_bench <N> <random 0/1> <seconds> [pattern: 0 one accumulator, 1 the GEMM's 3-accumulator order] [store warps 0-3]
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw64(uint32_t a) {
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

__device__ volatile int g_stop;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_mma2(int nn, int rnd, int pattern,
                                                                          long long iters, unsigned long long* out,
                                                                          int store_warps, unsigned long long* stores) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tslot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int e = threadIdx.x; e < 49152 / 4; e += blockDim.x) {
        uint32_t x = rnd ? (e * 2654435761u + blockIdx.x * 97u) ^ 0x5bd1e995u : 0u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        reinterpret_cast<uint32_t*>(sm)[e] = rnd ? x : 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nn >> 3) << 17) | ((256u >> 4) << 24);
    if (threadIdx.x >= 32 && (threadIdx.x >> 5) <= store_warps) {
        // competing shared-memory writes (16-byte stores into a separate 64 KB region)
        uint4* scratch = reinterpret_cast<uint4*>(sm + 49152);
        unsigned long long n = 0;
        const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        while (!g_stop) {
#pragma unroll 16
            for (int u = 0; u < 64; ++u) scratch[((threadIdx.x - 32) + 96 * u) & 4095] = v;
            n += 64;
        }
        atomicAdd(stores, n * 16);
    }
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(sm), b0 = a0 + 24576;
        uint32_t ph[2] = {0, 0};
        long long done = 0;
        for (long long it = 0; it < iters; ++it) {
            if (pattern == 0) {
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const uint64_t da = desc_sw64(a0 + 32 * (u & 1) + 8192 * ((u >> 1) & 1)), db = desc_sw64(b0 + 32 * (u & 1));
                    const uint32_t acc = u == 0 ? 0u : 1u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            } else {
                // the GEMM's pattern: 3 A slices (8 KB apart) x 3 B slices (5 KB apart), accumulators at
                // TMEM columns 0 / 160 / 320: per K32 step acc0, acc1, acc1, acc2, acc2, acc2
                const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0}, pd[6] = {0, 1, 1, 2, 2, 2};
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const int ks = (u / 6) & 1, m = u % 6;
                    const uint64_t da = desc_sw64(a0 + 8192 * pa[m] + 32 * ks), db = desc_sw64(b0 + 5120 * pb[m] + 32 * ks);
                    const uint32_t dt = tmem + (uint32_t)(nn * pd[m]);
                    const uint32_t acc = u < 6 ? 0u : 1u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            }
            const int s = (int)(it & 1);
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(&bar[s])), "h"((uint16_t)3) : "memory");
            done += 32;
            if (it >= 1) {
                const int q = s ^ 1;
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar[q])), "r"(ph[q]) : "memory");
                ph[q] ^= 1;
            }
        }
        const int q = (int)((iters - 1) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar[q])), "r"(ph[q]) : "memory");
        atomicAdd(out, (unsigned long long)done);
        g_stop = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    const int nn = argc > 1 ? atoi(argv[1]) : 160;
    const int rnd = argc > 2 ? atoi(argv[2]) : 0;
    const double secs = argc > 3 ? atof(argv[3]) : 1.0;
    const int pattern = argc > 4 ? atoi(argv[4]) : 0;
    const int store_warps = argc > 5 ? atoi(argv[5]) : 0;
    unsigned long long* dst;
    cudaMalloc(&dst, 8);
    int zero = 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 49152 + 65536 + 1024;
    cudaFuncSetAttribute(k_mma2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long long iters = 1000;
    float ms = 0;
    for (;;) {
        cudaMemset(d, 0, 8);
        cudaMemcpyToSymbol(g_stop, &zero, 4);
        cudaEventRecord(e0);
        k_mma2<<<sms & ~1, 128, smem>>>(nn, rnd, pattern, iters, d, store_warps, dst);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
        if (ms > 100) break;
        iters *= 4;
    }
    iters = (long long)(iters * (secs * 1e3 / ms));
    cudaMemset(d, 0, 8);
    cudaMemset(dst, 0, 8);
    cudaMemcpyToSymbol(g_stop, &zero, 4);
    cudaEventRecord(e0);
    k_mma2<<<sms & ~1, 128, smem>>>(nn, rnd, pattern, iters, d, store_warps, dst);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long mm = 0, sb = 0;
    cudaMemcpy(&mm, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&sb, dst, 8, cudaMemcpyDeviceToHost);
    // MACs per pair MMA: 256 x N x 32 ; per SM per cycle at the measured clock is computed by the caller
    const double macs = (double)mm * 256 * nn * 32;
    printf("{\"pattern\": %d, \"N\": %d, \"random\": %d, \"store_warps\": %d, \"ms\": %.1f, \"pair_mmas\": %llu, \"tops\": %.1f, \"smem_store_GBps_per_SM\": %.1f}\n",
           pattern, nn, rnd, store_warps, ms, mm, 2 * macs / (ms * 1e-3) / 1e12, sb / (ms * 1e-3) / sms / 1e9);
    return 0;
}

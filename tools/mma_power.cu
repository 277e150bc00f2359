// mma_power.cu -- microbenchmark: sustained tcgen05.mma throughput and SM clock
// under the 1 kW power cap, per MMA kind and operand data.  Not part of the
// library: it answers "which tensor-core arithmetic does the most fp32-class
// work per joule on this B200" before a precision scheme is chosen.
//
// One CTA per SM; A (128 x 128 B) and B (256 x 128 B) tiles sit in shared memory
// (SWIZZLE_128B, K-major) filled once with the chosen data; one thread issues
// MMAs M=128, N=256 over the 4 K-steps of the 128-byte rows back to back into a
// TMEM accumulator, committing every 64 MMAs with at most 2 commits in flight.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_power tools/mma_power.cu -lcuda
//   ./mma_power <mode> <seconds>
//   ./mma_power <mode> <seconds> [N]
// modes: 0 f16 gaussian   1 f16 "lo" split residues   2 f16 zeros   3 bf16 gaussian
//        4 s8 uniform [-127,127]   5 s8 zeros   6 e4m3 gaussian   7 s8 small [-8,8]
//        8 s8 uniform [-64,63]   9 s8 uniform [-32,31]
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ float gauss(uint32_t k) {  // Box-Muller from two hashes
    float u1 = (hash32(2 * k) + 1.f) * 2.3283064e-10f, u2 = hash32(2 * k + 1) * 2.3283064e-10f;
    return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}

__global__ void __launch_bounds__(128, 1) k_mma(int mode, int nn, long long iters, unsigned long long* out_mmas) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    uint8_t* A = sm;              // 128 rows x 128 B
    uint8_t* B = sm + 16384;      // 256 rows x 128 B
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    // fill 48 KB with the mode's data (layout irrelevant for power: any bytes)
    for (int e = tid; e < 49152 / 2; e += blockDim.x) {
        uint32_t key = blockIdx.x * 65536u + e;
        uint16_t v = 0;
        float g = gauss(key);
        switch (mode) {
            case 0: { __half h = __float2half_rn(g); v = *reinterpret_cast<uint16_t*>(&h); } break;
            case 1: { float x = g * 1024.f; __half h = __float2half_rn(x); __half l = __float2half_rn(x - __half2float(h));
                      v = *reinterpret_cast<uint16_t*>(&l); } break;
            case 2: v = 0; break;
            case 3: { __nv_bfloat16 h = __float2bfloat16_rn(g); v = *reinterpret_cast<uint16_t*>(&h); } break;
            case 4: { uint32_t h = hash32(key * 7 + 3); int8_t a = (int8_t)((int)(h % 255) - 127), b = (int8_t)((int)((h >> 8) % 255) - 127);
                      v = (uint16_t)(uint8_t)a | ((uint16_t)(uint8_t)b << 8); } break;
            case 5: v = 0; break;
            case 6: { __nv_fp8_e4m3 a(g), b(gauss(key + 77777777u)); v = (uint16_t)a.__x | ((uint16_t)b.__x << 8); } break;
            case 7: { uint32_t h = hash32(key * 7 + 3); int8_t a = (int8_t)((int)(h % 17) - 8), b = (int8_t)((int)((h >> 8) % 17) - 8);
                      v = (uint16_t)(uint8_t)a | ((uint16_t)(uint8_t)b << 8); } break;
            case 8: { uint32_t h = hash32(key * 7 + 3); int8_t a = (int8_t)((int)(h % 128) - 64), b = (int8_t)((int)((h >> 8) % 128) - 64);
                      v = (uint16_t)(uint8_t)a | ((uint16_t)(uint8_t)b << 8); } break;
            case 9: { uint32_t h = hash32(key * 7 + 3); int8_t a = (int8_t)((int)(h % 64) - 32), b = (int8_t)((int)((h >> 8) % 64) - 32);
                      v = (uint16_t)(uint8_t)a | ((uint16_t)(uint8_t)b << 8); } break;
        }
        reinterpret_cast<uint16_t*>(sm)[e] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    uint32_t idesc;
    const bool i8 = mode == 4 || mode == 5 || mode >= 7;
    const bool f8 = mode == 6;
    if (i8) idesc = (2u << 4) | (1u << 7) | (1u << 10);   // S32 <- S8 x S8
    else if (f8) idesc = (1u << 4);                        // F32 <- E4M3 x E4M3
    else idesc = (1u << 4) | ((mode == 3 ? 1u : 0u) << 7) | ((mode == 3 ? 1u : 0u) << 10);  // F32 <- F16/BF16
    idesc |= ((uint32_t)nn >> 3) << 17;
    idesc |= (128u >> 4) << 24;
    if (tid == 0) {
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
        uint32_t ph[2] = {0, 0};
        long long done = 0;
        for (long long it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t da = desc_sw128(a0 + 32 * k), db = desc_sw128(b0 + 32 * k);
                    const uint32_t acc = (u == 0 && k == 0) ? 0u : 1u;
                    if (i8)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    else if (f8)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            }
            const int s = (int)(it & 1);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar[s]))
                         : "memory");
            done += 64;
            if (it >= 1) {  // wait for the commit before this one
                const int q = s ^ 1;
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&bar[q])), "r"(ph[q]) : "memory");
                ph[q] ^= 1;
            }
        }
        // drain the last commit
        const int q = (int)((iters - 1) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar[q])), "r"(ph[q]) : "memory");
        atomicAdd(out_mmas, (unsigned long long)done);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const double seconds = argc > 2 ? atof(argv[2]) : 3.0;
    const int nn = argc > 3 ? atoi(argv[3]) : 256;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 49152 + 1024;
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // calibrate
    long long iters = 2000;
    float ms = 0;
    for (;;) {
        cudaMemset(d, 0, 8);
        cudaEventRecord(e0);
        k_mma<<<sms, 128, smem>>>(mode, nn, iters, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
        if (ms > 200) break;
        iters *= 4;
    }
    iters = (long long)(iters * (seconds * 1e3 / ms));
    cudaMemset(d, 0, 8);
    cudaEventRecord(e0);
    k_mma<<<sms, 128, smem>>>(mode, nn, iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long mm = 0;
    cudaMemcpy(&mm, d, 8, cudaMemcpyDeviceToHost);
    const bool byte8 = mode >= 4;
    // MACs per MMA: 128 x 256 x K, K = 16 (16-bit) or 32 (8-bit)
    const double macs = (double)mm * 128 * nn * (byte8 ? 32 : 16);
    printf("{\"N\": %d, \"mode\": %d, \"ms\": %.1f, \"mmas\": %llu, \"tops\": %.1f, \"mma_per_us_per_sm\": %.3f, \"err\": \"%s\"}\n",
           nn, mode, ms, mm, 2 * macs / (ms * 1e-3) / 1e12, mm / (ms * 1e3) / sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

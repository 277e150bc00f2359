// tma_bench.cu -- microbenchmark: how many bytes per clock can one SM pull into
// shared memory through TMA, per copy shape (no MMA)?  Each CTA (one per SM)
// cycles a 4-deep ring of 24 KB stages over a private 2 MB region of an
// L2-resident buffer.  mode 0: one 3-D tensor box {256 B, 32 rows, 3 planes}
// (the GEMM's A stage); mode 1: three 2-D boxes {256 B, 32 rows}; mode 2: three
// 8 KB cp.async.bulk (non-tensor) copies; mode 3: 256 threads issue 16-byte
// cp.async (LDGSTS) copies of the same stages; mode 4: 256 threads load 16-byte
// vectors into registers (raw L2 -> SM read rate, no shared-memory write).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_bench tools/tma_bench.cu -lcuda
//   ./tma_bench <mode> [CTAs]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) k_tma(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m2,
                                               const uint8_t* src, int mode, long long iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    __shared__ uint64_t bar[4];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long c0 = clock64();
    uint32_t ph[4] = {0, 0, 0, 0};
    const int64_t region = (int64_t)blockIdx.x * (2 << 20);  // 2 MB per CTA: 85 stages of 24 KB
    for (long long it = 0; it < iters; ++it) {
        const int s = (int)(it & 3);
        if (it >= 4) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(ph[s]) : "memory");
            ph[s] ^= 1;
        }
        const uint32_t dst = smem_u32(sm + s * 24576), mb = smem_u32(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(24576) : "memory");
        const int64_t off = region + (it % 85) * 24576;   // bytes into the buffer
        const int32_t row = (int32_t)(off / 256);
        if (mode == 0) {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                         ::"r"(dst), "l"(&m3), "r"(mb), "r"(0), "r"(row / 3), "r"(0) : "memory");
        } else if (mode == 1) {
            for (int p = 0; p < 3; ++p)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(dst + 8192 * p), "l"(&m2), "r"(mb), "r"(0), "r"(row + 32 * p) : "memory");
        } else {
            for (int p = 0; p < 3; ++p)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(dst + 8192 * p), "l"(src + off + 8192 * p), "r"(8192), "r"(mb) : "memory");
        }
    }
    for (int s = 0; s < 4; ++s) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(ph[s]) : "memory");
    }
    atomicAdd(cyc, (unsigned long long)(clock64() - c0));
}

__global__ void __launch_bounds__(256, 1) k_lsu(const uint8_t* src, int mode, long long iters,
                                                unsigned long long* cyc, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    const long long c0 = clock64();
    const int64_t region = (int64_t)blockIdx.x * (2 << 20);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (long long it = 0; it < iters; ++it) {
        const int s = (int)(it & 3);
        const int64_t off = region + (it % 85) * 24576;
        if (mode == 3) {
            for (int c = threadIdx.x; c < 24576 / 16; c += 256) {
                const uint32_t d = smem_u32(sm + s * 24576 + 16 * c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + off + 16 * c) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 3;" ::: "memory");
        } else {
#pragma unroll 6
            for (int c = threadIdx.x; c < 24576 / 16; c += 256) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src + off) + c);
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(clock64() - c0));
    if (acc.x == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 2 && atoi(argv[2]) > 0 && atoi(argv[2]) < sms) sms = atoi(argv[2]);  // CTAs (one per SM)
    const size_t bytes = (size_t)sms * (2 << 20) + (1 << 20);
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    CUtensorMap m3, m2;
    const cuuint64_t rows = bytes / 256;
    cuuint64_t d3[3] = {256, rows / 3, 3}, s3[2] = {256, (rows / 3) * 256};
    cuuint32_t b3[3] = {256, 32, 3}, e3[3] = {1, 1, 1};
    fn(&m3, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d2[2] = {256, rows}, s2[1] = {256};
    cuuint32_t b2[2] = {256, 32}, e2[2] = {1, 1};
    fn(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 4 * 24576 + 1024;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8);
    const long long iters = 40000;
    cudaFuncSetAttribute(k_lsu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(cyc, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (mode <= 2) k_tma<<<sms, 32, smem>>>(m3, m2, buf, mode, iters, cyc);
        else k_lsu<<<sms, 256, smem>>>(buf, mode, iters, cyc, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double per_sm_cycles = (double)c / sms;
        printf("{\"mode\": %d, \"ms\": %.2f, \"bytes_per_clk_per_SM\": %.1f, \"aggregate_TBps\": %.2f, \"err\": \"%s\"}\n", mode, ms,
               iters * 24576.0 / per_sm_cycles, iters * 24576.0 * sms / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

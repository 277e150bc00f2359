// sos_gemm.cu -- the two tensor-core kernels of the step (tcgen05 + TMEM,
// operands fed by the bulk-copy engine through an mbarrier ring).
//
//   forward:  G = V V^T on upper-triangular 128x256
//            tiles; the epilogue reduces every G_ij straight into
//            coef[rank(alpha_i + alpha_j)] (weight 2 off the diagonal, 1 on it),
//            so the N x N Gram matrix never reaches HBM.
//   backward (gradient of Eq. 2):      grad = 4 R V, R_ij = res[rank(alpha_i+alpha_j)]
//            read as split tiles of R, V^T as the B operand.
//
// fp32-class accuracy: every fp32 operand x is stored scaled by a power of two s
// as x*s = hi + lo (fp16 each, ~22 significant bits); each tile accumulates
//   A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T          (3 kind::f16 MMAs, fp32 in TMEM)
// and the epilogue divides the scales out.  The dropped A_lo B_lo^T term is
// O(2^-22) relative.
//
// Warp roles (320 threads, 1 CTA per SM, persistent over a static tile list):
//   warp 0      one lane issues the bulk copies (A 16 KB + B 32 KB per stage)
//   warp 1      allocates 512 TMEM columns; one lane issues tcgen05.mma
//   warps 2..9  epilogue: drain each K-segment accumulator (tcgen05.ld) into
//               fp32 register sums, then scatter / store the finished tile.
//               TMEM is double-buffered (2 x 256 columns) so draining segment
//               s overlaps the MMAs of segment s+1.
#include "sm100_ptx.cuh"
#include "sos_internal.cuh"

namespace sos {

struct GemmArgs {
    const uint8_t* A;
    const uint8_t* B;
    int64_t a_rows;  // rows_total of the A S-layout
    int64_t b_rows;  // rows_total of the B S-layout
    int num_kb;      // K-blocks of 32
    const TileCoord* tiles;
    int ntiles;
    const Scalars* scal;
    int64_t N;   // valid rows (monomials)
    int64_t Np;  // padded rows
    const uint32_t* pt;  // forward: pair-rank table
    float* coef;         // forward: output coefficients
    float* grad;         // backward: output N x r
    int64_t r;           // backward: columns of grad
    unsigned long long* progress;  // K-skew counter (zeroed before the launch)
};

constexpr uint32_t kSmemBytes = kStages * kStageBytes + 256 + 1024;

template <bool kFwd>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm(const GemmArgs args) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment of the shared-window address (SWIZZLE_128B atoms)
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        // ------------------------------------------------------- producer --
        if (lane == 0) {
            // Bounded K-skew: every kSkewEpoch K-blocks the producer publishes its
            // progress and does not run more than kSkewLag epochs ahead of the grid,
            // so the CTAs of a wave stream the same K-slabs of their shared panels
            // through L2 instead of whole panels (cooperative launch: all resident).
            int stage = 0;
            uint32_t phase = 0;
            int64_t g = 0;  // K-blocks issued by this CTA
            const unsigned long long G = gridDim.x;
            for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
                const TileCoord tc = args.tiles[tile];
                const uint8_t* srcA = args.A + (int64_t)tc.a * kBlockM * 128;
                const uint8_t* srcB = args.B + (int64_t)tc.b * kBlockN * 128;
                for (int kb = 0; kb < args.num_kb; ++kb, ++g) {
                    if (g % kSkewEpoch == 0 && g > 0) {
                        const int64_t e = g / kSkewEpoch;  // epochs completed by this CTA
                        atomicAdd(args.progress, 1ull);
                        if (e >= kSkewLag) {
                            const unsigned long long need = G * (unsigned long long)(e - kSkewLag + 1);
                            while (ld_acquire_u64(args.progress) < need) __nanosleep(256);
                        }
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * kStageBytes;
                    mbar_arrive_expect_tx(&full[stage], kStageBytes);
                    bulk_g2s(sa, srcA + (int64_t)kb * args.a_rows * 128, kTileABytes, &full[stage]);
                    bulk_g2s(sa + kTileABytes, srcB + (int64_t)kb * args.b_rows * 128, kTileBBytes, &full[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
            atomicAdd(args.progress, 1ull << 32);  // done: never hold back the others
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer --
        // The K loop of a tile is cut into segments of kSegKB K-blocks; each
        // segment accumulates into one of the two TMEM buffers from zero and is
        // drained by the epilogue into fp32 registers (round-to-nearest adds),
        // bounding the number of in-TMEM accumulations per value.
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_f16_f32(kBlockM, kBlockN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
                for (int kb0 = 0; kb0 < args.num_kb; kb0 += kSegKB) {
                    const int kb1 = min(args.num_kb, kb0 + kSegKB);
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d = tbase + acc * kBlockN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(smem + stage * kStageBytes);
                        const uint32_t b0 = a0 + kTileABytes;
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const uint64_t ah = umma_desc_sw128(a0 + s * 32);
                            const uint64_t al = umma_desc_sw128(a0 + 64 + s * 32);
                            const uint64_t bh = umma_desc_sw128(b0 + s * 32);
                            const uint64_t bl = umma_desc_sw128(b0 + 64 + s * 32);
                            umma_f16(d, ah, bh, idesc, (kb != kb0 || s != 0) ? 1u : 0u);
                            umma_f16(d, ah, bl, idesc, 1u);
                            umma_f16(d, al, bh, idesc, 1u);
                        }
                        umma_commit(&empty[stage]);  // smem slot free once these MMAs finish
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                    umma_commit(&tfull[acc]);  // segment accumulator ready for the epilogue
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else {
        // -------------------------------------------------------- epilogue --
        // 8 warps: warp w reads TMEM lane quarter q = w % 4 (rows 32q..32q+31 of
        // the tile) and column half h (128 columns); each thread keeps its
        // 128 running sums in registers.
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        float scale;
        if (kFwd) {
            const float s = args.scal->s_v;
            scale = 1.f / (s * s);
        } else {
            scale = 4.f / (args.scal->s_r * args.scal->s_v);
        }
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
            const TileCoord tc = args.tiles[tile];
            const int64_t i = (int64_t)tc.a * kBlockM + q * 32 + lane;
            float sum[kEpiCols];
#pragma unroll
            for (int t = 0; t < kEpiCols; ++t) sum[t] = 0.f;
            for (int kb0 = 0; kb0 < args.num_kb; kb0 += kSegKB) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + acc * kBlockN + h * kEpiCols;
#pragma unroll
                for (int ch = 0; ch < kEpiCols / 32; ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tq + ch * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int t = 0; t < 32; ++t) sum[ch * 32 + t] += __uint_as_float(v[t]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            const int64_t cbase = (int64_t)tc.b * kBlockN + h * kEpiCols;
            if (kFwd) {
                const bool strictly_upper = (int64_t)tc.a * kBlockM + kBlockM - 1 < (int64_t)tc.b * kBlockN;
#pragma unroll
                for (int ch = 0; ch < kEpiCols / 32; ++ch) {
                    const int64_t c0 = cbase + ch * 32;
                    const uint4* prow = reinterpret_cast<const uint4*>(args.pt + (((c0 >> 5) * args.Np + i) << 5));
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint4 rk = __ldg(prow + u);
                        const uint32_t rr[4] = {rk.x, rk.y, rk.z, rk.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int t = u * 4 + e;
                            if (rr[e] == kInvalidRank) continue;
                            const int64_t j = c0 + t;
                            const float w = strictly_upper ? 2.f : (i < j ? 2.f : (i == j ? 1.f : 0.f));
                            if (w != 0.f) red_add_f32(args.coef + rr[e], w * scale * sum[ch * 32 + t]);
                        }
                    }
                }
            } else if (i < args.N) {
#pragma unroll
                for (int ch = 0; ch < kEpiCols / 32; ++ch) {
                    const int64_t c0 = cbase + ch * 32;
                    float* g = args.grad + i * args.r + c0;
                    if (c0 + 32 <= args.r && ((reinterpret_cast<uintptr_t>(g) & 15) == 0)) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            float4 o;
                            o.x = scale * sum[ch * 32 + 4 * u + 0];
                            o.y = scale * sum[ch * 32 + 4 * u + 1];
                            o.z = scale * sum[ch * 32 + 4 * u + 2];
                            o.w = scale * sum[ch * 32 + 4 * u + 3];
                            reinterpret_cast<float4*>(g)[u] = o;
                        }
                    } else {
#pragma unroll
                        for (int t = 0; t < 32; ++t)
                            if (c0 + t < args.r) g[t] = scale * sum[ch * 32 + t];
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

static void launch(const Plan& P, const GemmArgs& a, bool fwd, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(k_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        configured = true;
    }
    const int grid = a.ntiles < P.num_sms ? a.ntiles : P.num_sms;
    if (grid <= 0) return;
    cudaMemsetAsync(a.progress, 0, sizeof(unsigned long long), st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (skew waits)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (fwd) cudaLaunchKernelEx(&cfg, k_gemm<true>, a);
    else cudaLaunchKernelEx(&cfg, k_gemm<false>, a);
}

void launch_gemm_fwd(Plan& P, float* coef, cudaStream_t st) {
    GemmArgs a{};
    a.A = P.d_vs;
    a.B = P.d_vs;
    a.a_rows = P.idx->Np;
    a.b_rows = P.idx->Np;
    a.num_kb = (int)(P.rK / kBlockK);
    a.tiles = P.d_tiles_fwd;
    a.ntiles = P.ntiles_fwd;
    a.scal = P.d_scal;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.pt = P.idx->d_pt;
    a.coef = coef;
    a.progress = P.d_progress;
    LaunchScope ls(P, KK_GEMM_FWD, st);
    launch(P, a, true, st);
}

void launch_gemm_bwd(Plan& P, float* grad, cudaStream_t st) {
    GemmArgs a{};
    a.A = P.d_rs;
    a.B = P.d_vts;
    a.a_rows = P.idx->Np;
    a.b_rows = P.rN;
    a.num_kb = (int)(P.idx->Np / kBlockK);
    a.tiles = P.d_tiles_bwd;
    a.ntiles = P.ntiles_bwd;
    a.scal = P.d_scal;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.grad = grad;
    a.r = P.r;
    a.progress = P.d_progress + 1;
    LaunchScope ls(P, KK_GEMM_BWD, st);
    launch(P, a, false, st);
}

}  // namespace sos

// sos_gemm2.cu -- the two tensor-core kernels of the step on CTA PAIRS
// (tcgen05 cta_group::2, UMMA M = 256 split over the two SMs of a cluster).
//
//   forward:  G = V V^T on upper-triangular 256x256
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
// A cluster of 2 CTAs owns one 256x256 output tile: CTA rank c holds rows
// [128c, 128c+128) of the A tile and of the B tile in its shared memory (16 KB
// each per 32-wide K-block), the leader (rank 0) issues tcgen05.mma.cta_group::2
// and each CTA's TMEM receives its 128 output rows x 256 columns.  Per SM this
// halves the B operand traffic (smem fill, L2 reads, smem reads by the tensor
// core) against one CTA per 128x256 tile.
//
// Warp roles (320 threads per CTA, 1 CTA per SM, persistent over a static tile list):
//   warp 0      one lane issues 2-SM TMA loads (A 16 KB + B 16 KB per stage),
//               completion counted on the leader's full barrier
//   warp 1      allocates 512 TMEM columns (pair-wide); the leader's lane 0 issues MMAs
//   warps 2..9  epilogue: drain each K-segment accumulator (tcgen05.ld) into
//               fp32 register sums, then scatter / store the finished tile;
//               the peer's warps release TMEM buffers on the leader's barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sm100_ptx.cuh"
#include "sos_internal.cuh"
#include "sos_split.cuh"

namespace sos {

struct Gemm2Args {
    int64_t a_rows;  // rows_total of the A S-layout
    int64_t b_rows;  // rows_total of the B S-layout
    int num_kb;      // K-blocks of 32
    const TileCoord* tiles;  // (256-row block, 256-col block)
    int ntiles;
    const Scalars* scal;
    int64_t N;
    int64_t Np;
    const uint32_t* pt;
    float* coef;
    float* grad;
    int64_t r;
    unsigned long long* progress;
    // kModeBwdUpdate: the optimiser step of PAPER.md:221, applied by the aux warps
    float* ring;  // per-CTA ring of 2 finished gradient tiles (128 x 256 fp32 each)
    float* V;
    float* m;
    float* v;
    int adam;
    float lr, b1, b2, lr_c1, inv_sqrt_c2, eps;
    // kModeFwd with Vsrc != nullptr: the aux warps pack V^T into VTS meanwhile
    const float* Vsrc;
    uint8_t* vts;
    int64_t rN;
    double stop_tol;  // kModeBwdUpdate: sos_opt_set_stop rule (0 = off)
};

constexpr int kModeFwd = 0;        // Gram tile -> coefficient scatter
constexpr int kModeBwdStore = 1;   // 4RV tile -> grad (sos_backward, sos_loss_grad)
constexpr int kModeBwdUpdate = 2;  // 4RV tile -> ring -> aux warps update V (and Adam moments)
constexpr int kRingTile = 128 * kBlockN;  // floats per ring slot

constexpr int kStages2 = 6;
constexpr uint32_t kHalfTileBytes = 128 * 128;  // 128 rows x 128 B
constexpr uint32_t kStage2Bytes = 2 * kHalfTileBytes;
constexpr uint32_t kAuxSmemBytes = 32 * 65 * 4;  // V tile staging of the aux warps' V^T pack
constexpr uint32_t kSmem2Bytes = kStages2 * kStage2Bytes + 512 + kAuxSmemBytes + 1024;
constexpr int kPairM = 256;

// aux warps: one optimiser step on a finished 128 x 256 gradient tile
// (coalesced: a warp covers 32 consecutive columns of one row per access)
__device__ __forceinline__ void update_tile(const Gemm2Args& a, const float* __restrict__ gt, int64_t row0,
                                            int64_t col0, int t) {
#pragma unroll 1
    for (int rr = 0; rr < 128; rr += 2) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int64_t i = row0 + rr + k;
            if (i >= a.N) continue;
            float gv[4], x[4], mm[4], vv[4];
            int64_t off[4];
            bool ok[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = t + 64 * e;
                ok[e] = col0 + c < a.r;
                off[e] = i * a.r + col0 + c;
                gv[e] = __ldcg(gt + (rr + k) * kBlockN + c);
                x[e] = ok[e] ? a.V[off[e]] : 0.f;
                if (a.adam) {
                    mm[e] = ok[e] ? a.m[off[e]] : 0.f;
                    vv[e] = ok[e] ? a.v[off[e]] : 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (!ok[e]) continue;
                if (a.adam) {
                    mm[e] = a.b1 * mm[e] + (1.f - a.b1) * gv[e];
                    vv[e] = a.b2 * vv[e] + (1.f - a.b2) * gv[e] * gv[e];
                    a.m[off[e]] = mm[e];
                    a.v[off[e]] = vv[e];
                    a.V[off[e]] = x[e] - a.lr_c1 * mm[e] / (sqrtf(vv[e]) * a.inv_sqrt_c2 + a.eps);
                } else {
                    a.V[off[e]] = x[e] - a.lr * gv[e];
                }
            }
        }
    }
}

// aux warps of the forward: VTS (V^T in the S-layout, K = row of V) for the
// backward that follows, one 32 (rows j) x 64 (columns c) tile at a time,
// transposed through shared memory; uses the scale s_v of this step's split.
__device__ __forceinline__ void pack_vts_tiles(const Gemm2Args& a, float (*buf)[65], int t) {
    const float s = a.scal->s_v;
    const int64_t ncb = a.rN / 64;
    const int64_t ntile = (a.Np / 32) * ncb;
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int64_t j0 = (tile / ncb) * 32, c0 = (tile % ncb) * 64;
        const int64_t c = c0 + t;
#pragma unroll 8
        for (int jj = 0; jj < 32; ++jj) {
            const int64_t j = j0 + jj;
            buf[jj][t] = (j < a.N && c < a.r) ? __ldg(a.Vsrc + j * a.r + c) * s : 0.f;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kAuxWarps));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int idx = t + 64 * k, cc = idx >> 2, q = idx & 3;
            float x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = buf[q * 8 + e][cc];
            store_split_row(a.vts + ((j0 >> 5) * a.rN + c0 + cc) * 128, c0 + cc, q, x);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kAuxWarps));
    }
}

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Gemm2Args args) {
    constexpr bool kFwd = kMode == kModeFwd;
    // converged (sos_opt_set_stop): the whole grid leaves before any barrier,
    // TMEM or cluster work, so V and the optimiser state stay as they are
    if (kMode == kModeBwdUpdate && descent_stopped(args.scal, args.stop_tol)) return;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStage2Bytes);
    uint64_t* empty = full + kStages2;
    uint64_t* tfull = empty + kStages2;
    uint64_t* tempty = tfull + 2;
    uint64_t* gready = tempty + 2;  // ring slot holds a finished gradient tile
    uint64_t* gfree = gready + 2;   // ring slot consumed by the aux warps
    uint32_t* tslot = reinterpret_cast<uint32_t*>(gfree + 2);
    float(*auxbuf)[65] = reinterpret_cast<float(*)[65]>(smem + kStages2 * kStage2Bytes + 512);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiWarps);  // epilogue warps of both CTAs
            mbar_init(&gready[a], kEpiWarps);
            mbar_init(&gfree[a], kAuxWarps);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
    }
    if (warp == 1) tmem_alloc_2sm(tslot, 512);
    tc_fence_before();
    cluster_sync();  // barrier inits + TMEM address visible pair-wide
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        // ------------------------------------------------------- producer --
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int64_t g = 0;
            const unsigned long long G = gridDim.x;
            for (int tile = cid; tile < args.ntiles; tile += ncl) {
                const TileCoord tc = args.tiles[tile];
                const int64_t rowA = (int64_t)tc.a * kPairM + rank * 128;
                const int64_t rowB = (int64_t)tc.b * kBlockN + rank * 128;
                for (int kb = 0; kb < args.num_kb; ++kb, ++g) {
                    // Bounded K-skew: every kSkewEpoch K-blocks the producer publishes its
                    // progress and waits (bounded) while it is more than kSkewLag epochs
                    // ahead of the grid, so the CTAs of a wave stream the same K-slabs of
                    // their shared panels through L2 instead of whole panels.
                    if (g % kSkewEpoch == 0 && g > 0) {
                        const int64_t e = g / kSkewEpoch;
                        atomicAdd(args.progress, 1ull);
                        if (e >= kSkewLag) {
                            const unsigned long long need = G * (unsigned long long)(e - kSkewLag + 1);
                            for (int spin = 0; spin < kSkewMaxSpin && ld_acquire_u64(args.progress) < need; ++spin)
                                __nanosleep(256);
                        }
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * kStage2Bytes;
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStage2Bytes);
                    tma_load_2d_2sm(sa, &tmA, &full[stage], 0, (int32_t)(kb * args.a_rows + rowA));
                    tma_load_2d_2sm(sa + kHalfTileBytes, &tmB, &full[stage], 0, (int32_t)(kb * args.b_rows + rowB));
                    if (++stage == kStages2) { stage = 0; phase ^= 1; }
                }
            }
            atomicAdd(args.progress, 1ull << 32);
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer --
        if (leader && lane == 0) {
            constexpr uint32_t idesc = umma_idesc_f16_f32(kPairM, kBlockN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = cid; tile < args.ntiles; tile += ncl) {
                for (int kb0 = 0; kb0 < args.num_kb; kb0 += kSegKB) {
                    const int kb1 = min(args.num_kb, kb0 + kSegKB);
                    mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d = tbase + acc * kBlockN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(smem + stage * kStage2Bytes);
                        const uint32_t b0 = a0 + kHalfTileBytes;
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const uint64_t ah = umma_desc_sw128(a0 + s * 32);
                            const uint64_t al = umma_desc_sw128(a0 + 64 + s * 32);
                            const uint64_t bh = umma_desc_sw128(b0 + s * 32);
                            const uint64_t bl = umma_desc_sw128(b0 + 64 + s * 32);
                            umma_f16_2sm(d, ah, bh, idesc, (kb != kb0 || s != 0) ? 1u : 0u);
                            umma_f16_2sm(d, ah, bl, idesc, 1u);
                            umma_f16_2sm(d, al, bh, idesc, 1u);
                        }
                        umma_commit_2sm(&empty[stage], 0x3);  // both CTAs' smem slots free
                        if (++stage == kStages2) { stage = 0; phase ^= 1; }
                    }
                    umma_commit_2sm(&tfull[acc], 0x3);  // both CTAs' epilogues may drain
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // -------------------------------------------------------- epilogue --
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
        int it = 0;
        for (int tile = cid; tile < args.ntiles; tile += ncl, ++it) {
            const TileCoord tc = args.tiles[tile];
            const int64_t i = (int64_t)tc.a * kPairM + rank * 128 + q * 32 + lane;
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
                if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            const int64_t cbase = (int64_t)tc.b * kBlockN + h * kEpiCols;
            if (kFwd) {
                // rows [a*256, a*256+256) vs cols [b*256, b*256+256): off the diagonal iff b > a
                const bool strictly_upper = tc.b > tc.a;
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
            } else if (kMode == kModeBwdUpdate) {
                // hand the finished tile to the aux warps through the per-CTA ring
                const int slot = it & 1;
                mbar_wait(&gfree[slot], ((it >> 1) & 1) ^ 1);
                float4* gr = reinterpret_cast<float4*>(args.ring + ((int64_t)blockIdx.x * 2 + slot) * kRingTile +
                                                       (q * 32 + lane) * kBlockN + h * kEpiCols);
#pragma unroll
                for (int u = 0; u < kEpiCols / 4; ++u)
                    gr[u] = make_float4(scale * sum[4 * u], scale * sum[4 * u + 1], scale * sum[4 * u + 2],
                                        scale * sum[4 * u + 3]);
                __threadfence_block();
                __syncwarp();
                if (lane == 0) mbar_arrive(&gready[slot]);
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
    } else if (kMode == kModeFwd) {
        // ----------------------------------------------------------- aux --
        if (args.Vsrc) pack_vts_tiles(args, auxbuf, threadIdx.x - 32 * (2 + kEpiWarps));
    } else if (kMode == kModeBwdUpdate) {
        // ----------------------------------------------------------- aux --
        // optimiser step on tile t while the tensor cores work on tile t+1
        const int t = threadIdx.x - 32 * (2 + kEpiWarps);  // 0..63
        int it = 0;
        for (int tile = cid; tile < args.ntiles; tile += ncl, ++it) {
            const TileCoord tc = args.tiles[tile];
            const int slot = it & 1;
            mbar_wait(&gready[slot], (it >> 1) & 1);
            update_tile(args, args.ring + ((int64_t)blockIdx.x * 2 + slot) * kRingTile,
                        (int64_t)tc.a * kPairM + rank * 128, (int64_t)tc.b * kBlockN, t);
            __syncwarp();
            if (lane == 0) mbar_arrive(&gfree[slot]);
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();  // all MMAs consumed and both epilogues done before freeing TMEM
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm(tbase, 512);
    }
}

// ------------------------------------------------------------------ host --
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// S-layout viewed as a 2-D byte array [kb * rows_total + row][128]; a box of
// 128 rows x 128 bytes is one contiguous, pre-swizzled 16 KB half tile.
bool make_split_tmap(void* map_out, const uint8_t* base, int64_t rows_total, int64_t num_kb) {
    CUtensorMap* map = reinterpret_cast<CUtensorMap*>(map_out);
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {128, (cuuint64_t)(rows_total * num_kb)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int kMode>
static cudaError_t launch2(const Plan& P, const CUtensorMap& ma, const CUtensorMap& mb, const Gemm2Args& a,
                           cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_gemm2<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes);
        configured = true;
    }
    int grid = 2 * a.ntiles < P.num_sms ? 2 * a.ntiles : P.num_sms;
    grid &= ~1;
    if (grid <= 0) return cudaSuccess;
    cudaMemsetAsync(a.progress, 0, sizeof(unsigned long long), st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kSmem2Bytes;
    cfg.stream = st;
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k_gemm2<kMode>, ma, mb, a);
}

static const CUtensorMap& tm(const uint8_t* raw) { return *reinterpret_cast<const CUtensorMap*>(raw); }

void launch_gemm2_fwd(Plan& P, float* coef, const float* V_for_vts, cudaStream_t st) {
    Gemm2Args a{};
    a.Vsrc = V_for_vts;
    a.vts = P.d_vts;
    a.rN = P.rN;
    a.r = P.r;
    a.a_rows = P.idx->Np;
    a.b_rows = P.idx->Np;
    a.num_kb = (int)(P.rK / kBlockK);
    a.tiles = P.d_tiles2_fwd;
    a.ntiles = P.ntiles2_fwd;
    a.scal = P.d_scal;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.pt = P.idx->d_pt;
    a.coef = coef;
    a.progress = P.d_progress;
    LaunchScope ls(P, KK_GEMM_FWD, st);
    launch2<kModeFwd>(P, tm(P.tmap_vs), tm(P.tmap_vs), a, st);
}

static Gemm2Args bwd_args(Plan& P) {
    Gemm2Args a{};
    a.a_rows = P.idx->Np;
    a.b_rows = P.rN;
    a.num_kb = (int)(P.idx->Np / kBlockK);
    a.tiles = P.d_tiles2_bwd;
    a.ntiles = P.ntiles2_bwd;
    a.scal = P.d_scal;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.r = P.r;
    a.progress = P.d_progress + 1;
    return a;
}

void launch_gemm2_bwd(Plan& P, float* grad, cudaStream_t st) {
    Gemm2Args a = bwd_args(P);
    a.grad = grad;
    LaunchScope ls(P, KK_GEMM_BWD, st);
    launch2<kModeBwdStore>(P, tm(P.tmap_rs), tm(P.tmap_vts), a, st);
}

// backward whose finished gradient tiles are consumed in the same kernel by the
// optimiser step (GD or Adam): the gradient never makes an HBM round trip.  The
// GEMM reads the packed copy VTS, never V, so updating V in place is safe.
void launch_gemm2_bwd_update(Plan& P, float* V, cudaStream_t st) {
    Gemm2Args a = bwd_args(P);
    a.ring = P.d_ring;
    a.V = V;
    a.stop_tol = P.stop_tol;
    a.lr = P.lr;
    a.adam = P.opt_kind == 1;
    if (a.adam) {
        const double c1 = 1.0 - pow((double)P.b1, (double)P.t);
        const double c2 = 1.0 - pow((double)P.b2, (double)P.t);
        a.m = P.d_m;
        a.v = P.d_v;
        a.b1 = P.b1;
        a.b2 = P.b2;
        a.eps = P.eps;
        a.lr_c1 = (float)(P.lr / c1);
        a.inv_sqrt_c2 = (float)(1.0 / sqrt(c2));
    }
    LaunchScope ls(P, KK_GEMM_BWD, st);
    launch2<kModeBwdUpdate>(P, tm(P.tmap_rs), tm(P.tmap_vts), a, st);
}

}  // namespace sos

// sos_gemmq.cu -- the two tensor-core kernels of the step on CTA PAIRS
// (tcgen05 cta_group::2, UMMA M = 256 split over the two SMs of a cluster),
// int8 slice arithmetic with exact s32 accumulation (sos_internal.cuh).
//
//   forward:  G = V V^T on upper-triangular 256 x 160
//            tiles; the epilogue reduces every G_ij straight into
//            coef[rank(alpha_i + alpha_j)] (weight 2 above the diagonal, 1 on it),
//            so the N x N Gram matrix never reaches HBM.
//   backward (gradient of Eq. 2):      grad = 4 R V, R_ij = res[rank(alpha_i+alpha_j)]
//            read as int8 slices of R, V^T as the B operand.
//
// Per 64-wide K-block each CTA stages its 128 A rows and 80 B rows, 3 slices
// each (24 KB + 15 KB, SWIZZLE_64B), in a 5-stage mbarrier ring filled by 2-SM
// TMA tensor loads; the leader issues, per 32-wide K step, the six slice
// products into three s32 TMEM accumulators (columns 0, 160, 320):
//     acc0 += a1 b1;  acc1 += a1 b2 + a2 b1;  acc2 += a1 b3 + a2 b2 + a3 b1.
// s32 accumulation is exact, so the accumulators are drained once per tile (or
// per kSegKBMax K-blocks for very long K) and combined in fp32 with the row
// scales: value = u_i u_j (acc0 + acc1/256 + acc2/65536).
//
// Warp roles (384 threads per CTA, 1 CTA per SM, persistent over a static tile list):
//   warp 0      producer: the 2-SM TMA loads (completion on the leader's barrier)
//   warp 1      allocates 512 TMEM columns (pair-wide); in the leader CTA it issues
//               the MMAs.  Both run as whole warps over warp-uniform state and issue
//               from one elect.sync lane (a single-lane loop cost ~15 % of the
//               tensor pipe in R2UR / BRA.U.ANY sequences)
//   warps 2..9  epilogue: TMEM lane quarter (warp & 3) x column half (80 columns);
//               in sos_step / sos_descend they also apply the optimiser update to
//               the drained tile (and write the next step's V slices) while the
//               tensor cores work on the next tile
//   warps 10,11 aux: forward -> pack V^T slices for the backward that follows
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sm100_ptx.cuh"
#include "sos_internal.cuh"
#include "sos_slice.cuh"

namespace sos {

// Experiment build only (-DSOS_EXPERIMENTS): the wait-cycle counters and the
// traffic probes below compile away in the shipped library.
#ifdef SOS_EXPERIMENTS
constexpr bool kExperiments = true;
#define SOS_CLOCK() clock64()
// SOS_GEMM_TRACE=1: CTA 0 records %globaltimer at phase boundaries (slot k) and prints them
#define GEMM_MARK(k) do { if (args.trace && blockIdx.x == 0) { unsigned long long now_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_)); tmark_s[k] = now_; } } while (0)
#else
constexpr bool kExperiments = false;
#define SOS_CLOCK() 0ll
#define GEMM_MARK(k) do { } while (0)
#endif

struct GemmArgs {
    int64_t a_rows;   // rows_total of the A Q-layout
    int64_t b_rows;   // rows_total of the B Q-layout
    int num_kb;       // K-blocks of 64
    int seg_kb;       // K-blocks per exact s32 TMEM segment
    const TileCoord* tiles;  // 256 rows x nb (<= 160) columns each
    int ntiles;
    const unsigned* umaxA;  // row maxima (float bits) of the A operand rows
    const unsigned* umaxB;  // row maxima of the B operand rows
    int64_t N;
    int64_t Np;
    const uint32_t* pt;
    float* coef;
    Scalars* zero_scal;  // forward inside sos_descend: clear the loss accumulators first
    float* grad;
    int64_t r;
    unsigned long long* progress;
    int skew_epoch, skew_lag;  // bounded K-skew (K-blocks per epoch, epochs of lead)
    int skew_sleep;            // ns between polls of the progress counter
    unsigned long long* dbg;   // experiments: SOS_GEMM_STATS per-role wait cycles
    int trace;                 // experiments: SOS_GEMM_TRACE phase times of CTA 0
    int kserp;                 // walk K backwards on odd local tiles (L2 reuse across waves)
    int skip_red;              // experiments: SOS_FWD_SKIP (wrong results): forward REDs skipped on
                               // 1 = tiles touching the diagonal, 2 = all tiles
    int probe;                 // experiments: SOS_GEMM_PROBE (wrong results): 1 = K-blocks mod 8,
                               // 2 = also tile 0, 4 = 2 with B loaded only on the first ring pass
    // kModeBwdUpdate(Vtq): the optimiser step of PAPER.md:221, applied by the epilogue warps
    float* ring;  // per-CTA staging of the finished gradient tile (128 x 160 fp32, L2-resident)
    float* V;
    float* m;
    float* v;
    int adam;
    const Scalars* scal;
    const DevOpt* opt;  // optimiser parameters, step count t, stopping tolerance
    int use_stop;       // apply the sos_opt_set_stop rule
    // kModeBwdUpdate(Vtq) inside sos_descend (vq_next != nullptr): the update also
    // writes the int8 slices of the updated V (scale kHeadroom * vrow_cur) and the
    // exact row / column maxima of the updated V for the next step
    uint8_t* vq_next;
    int64_t rowsV, nkbV;
    const unsigned* vrow_cur;
    unsigned* vrow_next;
    unsigned* vcol_next;
    // kModeFwd with Vsrc != nullptr: the aux warps pack V^T slices meanwhile;
    // kModeBwdUpdateVtq: the update also writes the next step's
    // V^T slices (column scale kHeadroom * vcol)
    const float* Vsrc;
    uint8_t* vtq;
    int64_t rowsVT;
    int64_t nkbN;
    const unsigned* vcol;
    // kModeBwdUpdate(Vtq), last step of sos_solve_host: after the update of a tile is
    // stored, both CTAs of the pair add 1 to rowsig[tile.a / sig_blocks] (system
    // scope) so a copy stream can ship finished row chunks of V while the rest runs
    unsigned* rowsig;
    int sig_blocks;
    int sig_chunks;
};

// Adam / GD constants of this step, formed on the device from DevOpt
struct OptConsts {
    float lr, b1, b2, eps, lr_c1, inv_sqrt_c2;
};

constexpr int kModeFwd = 0;        // Gram tile -> coefficient scatter
constexpr int kModeBwdStore = 1;   // 4RV tile -> grad (sos_backward, sos_loss_grad)
constexpr int kModeBwdUpdate = 2;  // 4RV tile -> staged -> epilogue warps update V (and Adam moments)
constexpr int kModeBwdUpdateVtq = 3;  // same, also writing the next step's V^T slices (separate
                                      // instantiation: the extra code costs registers otherwise)
constexpr int kRingTile = 128 * kTileN;  // floats per ring slot

constexpr int kStages = 5;
constexpr uint32_t kASliceBytes = 128 * 64;        // 8 KB
constexpr uint32_t kBSliceBytes = kHalfN * 64;     // 5 KB
constexpr uint32_t kABytes = kSlices * kASliceBytes;
constexpr uint32_t kBBytes = kSlices * kBSliceBytes;
constexpr uint32_t kStageBytes = kABytes + kBBytes;  // 39936
constexpr uint32_t kBarBytes = 256;
constexpr uint32_t kAuxSmemBytes = 64 * 65 * 4;    // V tile staging of the aux warps' V^T pack
constexpr uint32_t kColScaleBytes = 2 * kTileN * 4; // the epilogue's column scales, double-buffered by tile
constexpr uint32_t kSmemBytes = kStages * kStageBytes + kBarBytes + kAuxSmemBytes + kColScaleBytes + 1024;
constexpr float kInv256 = 1.f / 256.f;
constexpr float kInv65536 = 1.f / 65536.f;

constexpr int kQRows = 16;  // rows per staged batch of the update

// The optimiser step on a finished 128 x 160 gradient tile (ring slot gt) by the
// 8 epilogue warps, right after they drained it (the tensor cores already work
// on the next tile).  Batches of 16 rows: warp w owns rows 2w, 2w+1 of a batch,
// lane l the columns l + 32e (e < 5): every access is a coalesced row segment,
// all 40 loads of a thread are in flight together, and a thread keeps the same
// 5 columns for the whole tile (column maxima in registers).  Inside
// sos_descend (vq_next) the new rows are staged in shared memory and sliced
// into the next step's VQ with the scale kHeadroom * max|row of the current V|,
// valid while the row maximum stays in [1/2, 2] of the old one (k_descend_fixup
// re-slices the rare rows that leave that window, see sos_pointwise.cu).
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kStageLd = kTileN + 4;  // staged row pitch (floats): column reads hit distinct banks
template <bool kVtq>
__device__ __forceinline__ void update_tile_epi(const GemmArgs& a, const OptConsts& o, const float* __restrict__ gt,
                                                int64_t row0, int64_t col0, int w, int lane, float* stage) {
    constexpr int kE = kTileN / 32;  // columns per lane
    const bool q = a.vq_next != nullptr;
    float cm[kE];
#pragma unroll
    for (int e = 0; e < kE; ++e) cm[e] = 0.f;
#pragma unroll 1
    for (int rb = 0; rb < 128; rb += kQRows) {
        if (row0 + rb >= a.N) break;
        float gv[2][kE], x[2][kE], mm[2][kE], vv[2][kE];
        int64_t ro[2];  // element offset of (row, col0 + lane); column e adds 32 e
        bool ok[2][kE];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int rr = rb + 2 * w + k;
            const int64_t i = row0 + rr;
            ro[k] = i * a.r + col0 + lane;
#pragma unroll
            for (int e = 0; e < kE; ++e) {
                const int c = lane + 32 * e;
                ok[k][e] = col0 + c < a.r && i < a.N;
                gv[k][e] = ok[k][e] ? __ldcg(gt + rr * kTileN + c) : 0.f;
                x[k][e] = ok[k][e] ? __ldcs(a.V + ro[k] + 32 * e) : 0.f;
                if (a.adam) {
                    mm[k][e] = ok[k][e] ? __ldcs(a.m + ro[k] + 32 * e) : 0.f;
                    vv[k][e] = ok[k][e] ? __ldcs(a.v + ro[k] + 32 * e) : 0.f;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float m = 0.f;
#pragma unroll
            for (int e = 0; e < kE; ++e) {
                float xn = 0.f;
                if (ok[k][e]) {
                    if (a.adam) {
                        mm[k][e] = o.b1 * mm[k][e] + (1.f - o.b1) * gv[k][e];
                        vv[k][e] = o.b2 * vv[k][e] + (1.f - o.b2) * gv[k][e] * gv[k][e];
                        xn = x[k][e] - o.lr_c1 * mm[k][e] / (sqrtf(vv[k][e]) * o.inv_sqrt_c2 + o.eps);
                        __stcs(a.m + ro[k] + 32 * e, mm[k][e]);
                        __stcs(a.v + ro[k] + 32 * e, vv[k][e]);
                    } else {
                        xn = x[k][e] - o.lr * gv[k][e];
                    }
                    __stcs(a.V + ro[k] + 32 * e, xn);
                }
                if (q) {
                    stage[(2 * w + k) * kStageLd + lane + 32 * e] = xn;
                    const float ax = fabsf(xn);
                    m = fmaxf(m, ax);
                    cm[e] = fmaxf(cm[e], ax);
                }
            }
            if (q) {
#pragma unroll
                for (int s = 16; s; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
                const int64_t i = row0 + rb + 2 * w + k;
                if (lane == 0 && i < a.N && m > 0.f) atomicMax(a.vrow_next + i, __float_as_uint(m));
            }
        }
        if (!q) continue;
        asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads));  // batch staged
        const int t = w * 32 + lane;
        if (t < kQRows * (kTileN / 16)) {  // task = (row, 16-column chunk)
            const int rr = t / (kTileN / 16), cq = t - rr * (kTileN / 16);
            const int64_t i = row0 + rb + rr, k0 = col0 + 16 * cq;
            if (i < a.N && k0 < a.r) {
                float xs[16];
                const float4* s4 = reinterpret_cast<const float4*>(stage + rr * kStageLd + 16 * cq);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const float4 f = s4[q4];
                    xs[4 * q4] = f.x; xs[4 * q4 + 1] = f.y; xs[4 * q4 + 2] = f.z; xs[4 * q4 + 3] = f.w;
                }
                const float um = kHeadroom * __uint_as_float(__ldg(a.vrow_cur + i));
                uint4 qq[3];
                slice16(xs, slice_scale(__float_as_uint(um)), qq);
                store_q16(a.vq_next, k0 >> 6, i, (int)((k0 >> 4) & 3), a.nkbV, a.rowsV, qq);
            }
        }
        const int tv = kEpiThreads - 1 - t;  // VTQ task of this thread (threads 96.. ; 160 tasks)
        if (kVtq && tv < kTileN && col0 + tv < a.r) {
            // VTQ row k = col0 + tv: the batch's 16 rows are one 16-value K-chunk of it
            const int64_t k = col0 + tv, i0 = row0 + rb;
            float xs[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) xs[e] = stage[e * kStageLd + tv];
            const float uc = kHeadroom * __uint_as_float(__ldg(a.vcol + k));
            uint4 qq[3];
            slice16(xs, slice_scale(__float_as_uint(uc)), qq);
            store_q16(a.vtq, i0 >> 6, k, (int)((i0 >> 4) & 3), a.nkbN, a.rowsVT, qq);
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads));  // stage free
    }
    if (q) {
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const int c = lane + 32 * e;
            if (col0 + c < a.r && cm[e] > 0.f) atomicMax(a.vcol_next + col0 + c, __float_as_uint(cm[e]));
        }
    }
}

__device__ __forceinline__ OptConsts opt_consts(const DevOpt* p) {
    const DevOpt o = *p;
    OptConsts oc;
    oc.lr = o.lr;
    oc.b1 = o.b1;
    oc.b2 = o.b2;
    oc.eps = o.eps;
    oc.lr_c1 = o.lr_c1;  // advance_step (k_step_begin) formed them for this step
    oc.inv_sqrt_c2 = o.inv_sqrt_c2;
    return oc;
}

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_gemmq(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
    constexpr bool kFwd = kMode == kModeFwd;
    constexpr bool kUpd = kMode == kModeBwdUpdate || kMode == kModeBwdUpdateVtq;
    extern __shared__ uint8_t smem_raw[];
#ifdef SOS_EXPERIMENTS
    __shared__ unsigned long long tmark_s[10];
    __shared__ unsigned long long wend_s[kGemmThreads / 32];
    if (threadIdx.x < 10) tmark_s[threadIdx.x] = 0;
    if (threadIdx.x == 0) GEMM_MARK(0);
#endif
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
    float(*auxbuf)[65] = reinterpret_cast<float(*)[65]>(smem + kStages * kStageBytes + kBarBytes);
    float* colscale = reinterpret_cast<float*>(smem + kStages * kStageBytes + kBarBytes + kAuxSmemBytes);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 2 * kEpiWarps);  // epilogue warps of both CTAs
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
    if (threadIdx.x == 0) GEMM_MARK(1);
    // launched with programmatic stream serialization (split steps), the setup
    // above overlapped the previous kernel's tail; its results are visible from here
    griddep_wait();
    if (threadIdx.x == 0) GEMM_MARK(2);
    // converged (sos_opt_set_stop): no CTA touches V or the optimiser state
    const bool stopped = kUpd && descent_stopped(args.scal, args.opt, args.use_stop);
    if (stopped && args.rowsig && blockIdx.x == 0)  // nothing changes: release every chunk at once
        for (int c = threadIdx.x; c < args.sig_chunks; c += blockDim.x) atomicExch(args.rowsig + c, kSigReleased);
    if (kFwd && args.zero_scal && blockIdx.x == 0 && threadIdx.x == 0) {
        args.zero_scal->loss = 0.0;  // the residual that follows accumulates the new loss
        args.zero_scal->pnorm2 = 0.0;
    }

    if (stopped) {
        // grid-uniform: straight to the teardown
    } else if (warp == 0) {
        // ------------------------------------------------------- producer --
        // whole warp (warp-uniform loop state), one elected lane issues
        {
            int stage = 0;
            uint32_t phase = 0;
            int64_t g = 0;
            const unsigned long long G = gridDim.x;
            int it = 0;
            for (int tile = cid; tile < args.ntiles; tile += ncl, ++it) {
                const TileCoord tc = args.tiles[tile];
                // serpentine K: consecutive waves share their A panels (grouped raster), so
                // every other tile walks K backwards and starts on the slabs the previous
                // wave loaded last, still in L2 (-1.4 % step time, profiles/r1_l2_probes.md)
                const bool rev = args.kserp && (it & 1);
                const int32_t rowA = tc.a * kPairM + (int)rank * 128;
                const int32_t rowB = tc.c0 + (int)rank * (tc.nb >> 1);  // each CTA supplies nb/2 B rows
                for (int kb = 0; kb < args.num_kb; ++kb, ++g) {
                    // Bounded K-skew: every kSkewEpoch K-blocks the producer publishes its
                    // progress and waits (bounded) while it is more than kSkewLag epochs
                    // ahead of the grid, so the CTAs of a wave stream the same K-slabs of
                    // their shared panels through L2 instead of whole panels.
                    if (g % args.skew_epoch == 0 && g > 0) {
                        const int64_t e = g / args.skew_epoch;
                        if (lane == 0) atomicAdd(args.progress, 1ull);
                        if (e >= args.skew_lag) {
                            const unsigned long long need = G * (unsigned long long)(e - args.skew_lag + 1);
                            const long long c0 = SOS_CLOCK();
                            if (lane == 0)
                                for (int spin = 0; spin < kSkewMaxSpin && ld_acquire_u64(args.progress) < need; ++spin)
                                    if (args.skew_sleep) __nanosleep(args.skew_sleep);
                            __syncwarp();
                            if (kExperiments && args.dbg && lane == 0) atomicAdd(args.dbg + 0, (unsigned long long)(SOS_CLOCK() - c0));
                        }
                    }
                    {
                        const long long c0 = SOS_CLOCK();
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (kExperiments && args.dbg && lane == 0) atomicAdd(args.dbg + 1, (unsigned long long)(SOS_CLOCK() - c0));
                    }
                    if (elect_one()) {
                        uint8_t* sa = smem + stage * kStageBytes;
                        const bool skipB = kExperiments && args.probe == 4 && g >= kStages;
                        if (leader) mbar_arrive_expect_tx(&full[stage], skipB ? 2 * kABytes : 2 * kStageBytes);
                        // the tensor maps view 4 consecutive 64-byte Q-rows as one 256-byte row
                        const int kq = kExperiments && args.probe ? (kb & 7) : rev ? args.num_kb - 1 - kb : kb;
                        const int32_t ra = kExperiments && args.probe >= 2 ? (int32_t)rank * 128 : rowA;
                        const int32_t rb = kExperiments && args.probe >= 2 ? (int32_t)rank * kHalfN : rowB;
                        tma_load_3d_2sm(sa, &tmA, &full[stage], 0, (int32_t)((kq * args.a_rows + ra) >> 2), 0);
                        if (!skipB)
                            tma_load_3d_2sm(sa + kABytes, &tmB, &full[stage], 0, (int32_t)((kq * args.b_rows + rb) >> 2), 0);
                    }
                    __syncwarp();
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
            if (lane == 0) {
                // done marker (releases any CTA still pacing itself); the last CTA to
                // finish resets the counter for the next launch (no memset per launch)
                const unsigned long long old = atomicAdd(args.progress, 1ull << 32);
                if ((old >> 32) + 1 == (unsigned long long)gridDim.x) atomicExch(args.progress, 0ull);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer --
        // the whole warp runs the loop (waits, descriptor arithmetic: warp-uniform
        // values in uniform registers); one elected lane issues the MMAs and
        // commits.  A single-lane loop spent ~15 % of the tensor pipe on issue.
        if (leader) {
            const long long t_start = SOS_CLOCK();
            const uint32_t d0 = tbase, d1 = tbase + kTileN, d2 = tbase + 2 * kTileN;
            // descriptor of stage 0, slice 0; other operands differ only in the
            // start-address field (bits 0-13, 16-byte units)
            const uint64_t desc0 = umma_desc_sw64(smem_u32(smem));
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_phase = 0;
            for (int tile = cid; tile < args.ntiles; tile += ncl) {
                const uint32_t idesc = umma_idesc_s8_s32(kPairM, args.tiles[tile].nb);
                for (int kb0 = 0; kb0 < args.num_kb; kb0 += args.seg_kb) {
                    const int kb1 = min(args.num_kb, kb0 + args.seg_kb);
                    {
                        const long long c0 = SOS_CLOCK();
                        mbar_wait_cluster(tempty, acc_phase ^ 1);
                        if (kExperiments && args.dbg && lane == 0) atomicAdd(args.dbg + 2, (unsigned long long)(SOS_CLOCK() - c0));
                    }
                    tc_fence_after();
                    for (int kb = kb0; kb < kb1; ++kb) {
                        {
                            const long long c0 = SOS_CLOCK();
                            mbar_wait(&full[stage], phase);
                            if (kExperiments && args.dbg && lane == 0) atomicAdd(args.dbg + 3, (unsigned long long)(SOS_CLOCK() - c0));
                        }
                        if (kExperiments && lane == 0 && tile == cid && kb == 0) GEMM_MARK(3);
                        tc_fence_after();
                        const uint64_t sd = desc0 + (uint64_t)((stage * kStageBytes) >> 4);
                        const uint64_t bd = sd + (kABytes >> 4);
                        const bool first = kb == kb0;
                        if (elect_one()) {
                            // per 32-wide K step (ks) the MMAs that share an A slice run back
                            // to back and take A from the tensor core's collector buffer after
                            // the first read (collector::a fill / use / lastuse)
#pragma unroll
                            for (int ks = 0; ks < 2; ++ks) {
                                const uint64_t k2 = (uint64_t)(ks * 2);  // +32 bytes
                                const uint64_t a1 = sd + k2, a2 = sd + (kASliceBytes >> 4) + k2,
                                               a3 = sd + (2 * kASliceBytes >> 4) + k2;
                                const uint64_t b1 = bd + k2, b2 = bd + (kBSliceBytes >> 4) + k2,
                                               b3 = bd + (2 * kBSliceBytes >> 4) + k2;
                                const uint32_t acc = (first && ks == 0) ? 0u : 1u;
                                umma_s8_2sm<1>(d0, a1, b1, idesc, acc);  // a1 read once, kept
                                umma_s8_2sm<2>(d1, a1, b2, idesc, acc);
                                umma_s8_2sm<3>(d2, a1, b3, idesc, acc);  // a1 released
                                umma_s8_2sm<1>(d1, a2, b1, idesc, 1u);   // a2 read once, kept
                                umma_s8_2sm<3>(d2, a2, b2, idesc, 1u);   // a2 released
                                umma_s8_2sm<0>(d2, a3, b1, idesc, 1u);
                            }
                            umma_commit_2sm(&empty[stage], 0x3);  // both CTAs' smem slots free
                        }
                        __syncwarp();
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) umma_commit_2sm(tfull, 0x3);  // both CTAs' epilogues may drain
                    if (kExperiments && lane == 0) GEMM_MARK(4);
                    __syncwarp();
                    acc_phase ^= 1;
                }
            }
            if (kExperiments && args.dbg && lane == 0) atomicAdd(args.dbg + 4, (unsigned long long)(SOS_CLOCK() - t_start));
        }
    } else if (warp < 2 + kEpiWarps) {
        // -------------------------------------------------------- epilogue --
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        OptConsts oc{};
        if (kUpd) oc = opt_consts(args.opt);
        uint32_t acc_phase = 0;
        int it = 0;
        for (int tile = cid; tile < args.ntiles; tile += ncl, ++it) {
            const TileCoord tc = args.tiles[tile];
            const int64_t i = (int64_t)tc.a * kPairM + rank * 128 + q * 32 + lane;
            // the tile's column scales u_j into shared memory while the MMAs run (one
            // load per column instead of a dependent L2 round trip per 4 columns in
            // every epilogue thread); double-buffered by tile parity: a thread can
            // reach tile k+2 only after every thread passed tile k+1's barrier
            float* cs = colscale + (it & 1) * kTileN;
            {
                const int et = (warp - 2) * 32 + lane;
                if (et < tc.nb) cs[et] = slice_unit(__ldg(args.umaxB + tc.c0 + et));
                asm volatile("bar.sync 3, %0;" ::"n"(kEpiThreads));
            }
            const float* csh = cs + h * kEpiCols;
            float sum[kEpiCols];
#pragma unroll
            for (int t = 0; t < kEpiCols; ++t) sum[t] = 0.f;
            const int ncol = min(kEpiCols, tc.nb - h * kEpiCols);  // this warp's live columns (<= 0: none)
            for (int kb0 = 0; kb0 < args.num_kb; kb0 += args.seg_kb) {
                mbar_wait(tfull, acc_phase);
                if (kExperiments && warp == 2 && lane == 0 && tile == cid && kb0 == 0) GEMM_MARK(5);
                tc_fence_after();
                const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + h * kEpiCols;
#pragma unroll
                for (int ch = 0; ch < kEpiCols / 16; ++ch) {
                    if (ch * 16 >= ncol) break;  // warp-uniform
                    uint32_t v0[16], v1[16], v2[16];
                    tmem_ld16(tq + ch * 16, v0);
                    tmem_ld16(tq + kTileN + ch * 16, v1);
                    tmem_ld16(tq + 2 * kTileN + ch * 16, v2);
                    tmem_ld_wait();
#pragma unroll
                    for (int t = 0; t < 16; ++t)
                        sum[ch * 16 + t] += fmaf((float)(int)v2[t], kInv65536,
                                                 fmaf((float)(int)v1[t], kInv256, (float)(int)v0[t]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty, 0);
                acc_phase ^= 1;
            }
            if (kExperiments && warp == 2 && lane == 0 && tile == cid) GEMM_MARK(8);
            const int64_t cbase = (int64_t)tc.c0 + h * kEpiCols;
            const float ui = slice_unit(__ldg(args.umaxA + i));
            if (kExperiments && warp == 2 && lane == 0 && tile == cid) GEMM_MARK(9);
            if (kFwd) {
                // rows [256a, 256a+256) vs cols [c0, c0+nb): all above the diagonal iff c0 >= 256a + 256
                const bool strictly_upper = (int64_t)tc.c0 >= (int64_t)tc.a * kPairM + kPairM;
                const bool skip = kExperiments && (args.skip_red == 2 || (args.skip_red == 1 && !strictly_upper));
                if (i < args.N && !skip) {
                    // 16-column chunks: live, inside N, and in the stored PT triangle (a
                    // later row block means j < i for all 16 columns: weight 0)
                    bool live[kEpiCols / 16];
#pragma unroll
                    for (int ch = 0; ch < kEpiCols / 16; ++ch) {
                        const int64_t c0 = cbase + ch * 16;
                        live[ch] = ch * 16 < ncol && c0 < args.N && (i >> 6) <= (c0 >> 6);
                    }
                    // the pair ranks of the next chunk are in flight while this one scatters
                    uint4 rk[2][4];
                    if (live[0]) {
                        const uint4* prow = reinterpret_cast<const uint4*>(args.pt + pt_entry(i, cbase));
#pragma unroll
                        for (int u = 0; u < 4; ++u) rk[0][u] = __ldg(prow + u);
                    }
#pragma unroll
                    for (int ch = 0; ch < kEpiCols / 16; ++ch) {
                        if (ch + 1 < kEpiCols / 16 && live[ch + 1]) {
                            const uint4* prow =
                                reinterpret_cast<const uint4*>(args.pt + pt_entry(i, cbase + (ch + 1) * 16));
#pragma unroll
                            for (int u = 0; u < 4; ++u) rk[(ch + 1) & 1][u] = __ldg(prow + u);
                        }
                        if (!live[ch]) continue;
                        const int64_t c0 = cbase + ch * 16;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint4 k4 = rk[ch & 1][u];
                            const uint32_t rr[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int t = u * 4 + e;
                                if (rr[e] == kInvalidRank) continue;
                                const int64_t j = c0 + t;
                                const float w = strictly_upper ? 2.f : (i < j ? 2.f : (i == j ? 1.f : 0.f));
                                if (w != 0.f)
                                    red_add_f32(args.coef + rr[e], w * ui * csh[ch * 16 + t] * sum[ch * 16 + t]);
                            }
                        }
                    }
                }
            } else if (kUpd) {
                // stage the finished tile (thread = row) in the ring, then update it
                // coalesced (thread = column) with all 8 epilogue warps
                float4* gr = reinterpret_cast<float4*>(args.ring + (int64_t)blockIdx.x * kRingTile +
                                                       (q * 32 + lane) * kTileN + h * kEpiCols);
                const float s4 = 4.f * ui;
#pragma unroll
                for (int u = 0; u < kEpiCols / 4; ++u)
                    gr[u] = make_float4(s4 * csh[4 * u] * sum[4 * u], s4 * csh[4 * u + 1] * sum[4 * u + 1],
                                        s4 * csh[4 * u + 2] * sum[4 * u + 2], s4 * csh[4 * u + 3] * sum[4 * u + 3]);
                __threadfence_block();
                asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads));  // whole tile in the ring
                update_tile_epi<kMode == kModeBwdUpdateVtq>(args, oc, args.ring + (int64_t)blockIdx.x * kRingTile,
                                (int64_t)tc.a * kPairM + rank * 128, (int64_t)tc.c0, warp - 2, lane,
                                reinterpret_cast<float*>(auxbuf));
                asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads));  // ring consumed
                if (args.rowsig && warp == 2 && lane == 0) {
                    __threadfence_system();
                    atomicAdd(args.rowsig + tc.a / args.sig_blocks, 1u);
                }
            } else {
                // gradient store (sos_backward, sos_loss_grad, split step).  A thread holds
                // one row, so direct stores would put 32 rows in every warp store; each
                // 16-column chunk goes through a per-warp shared-memory tile instead
                // (XOR-swizzled: conflict-free reads, 2-way writes) and leaves as two
                // full 64-byte row segments per warp store
                float* wbuf = &auxbuf[0][0] + (warp - 2) * 32 * 16;
                const float s4 = 4.f * ui;
                const int64_t row0 = (int64_t)tc.a * kPairM + rank * 128 + q * 32;
#pragma unroll
                for (int ch = 0; ch < kEpiCols / 16; ++ch) {
                    if (ch * 16 >= ncol) break;  // warp-uniform
#pragma unroll
                    for (int e = 0; e < 16; ++e) wbuf[lane * 16 + (e ^ (lane & 15))] = s4 * csh[ch * 16 + e] * sum[ch * 16 + e];
                    __syncwarp();
                    const int c = lane & 15;
                    const int64_t col = cbase + ch * 16 + c;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const int rr = 2 * k + (lane >> 4);
                        const int64_t row = row0 + rr;
                        if (row < args.N && col < args.r && ch * 16 + c < ncol)
                            args.grad[row * args.r + col] = wbuf[rr * 16 + (c ^ (rr & 15))];
                    }
                    __syncwarp();
                }
            }
        }
    } else if (kMode == kModeFwd) {
        // ----------------------------------------------------------- aux --
        // V^T slices for the backward that follows (hidden under the MMA loop)
        if (args.Vsrc) {
            const int t = threadIdx.x - 32 * (2 + kEpiWarps);
            const int64_t nkt = (args.rowsVT + 63) / 64;
            for (int64_t b = blockIdx.x; b < args.nkbN * nkt; b += gridDim.x)
                pack_vtq_tile<32 * kAuxWarps>(args.Vsrc, args.N, args.r, args.rowsVT, args.nkbN, args.vcol, args.vtq,
                                              b / nkt, (b % nkt) * 64, auxbuf, t);
        }
    }

    if (kExperiments && warp == 2 && lane == 0) GEMM_MARK(6);
#ifdef SOS_EXPERIMENTS
    if (args.trace && blockIdx.x < 2 && lane == 0) {  // per-warp end of the role loops, CTAs 0 and 1
        unsigned long long now_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));
        wend_s[warp] = now_;
    }
#endif
    tc_fence_before();
    __syncthreads();
    // all MMAs consumed and both epilogues' TMEM reads done before freeing TMEM
    // (relaxed: no need to wait for the epilogues' global REDs / stores here)
    cluster_sync_relaxed();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm(tbase, 512);
    }
#ifdef SOS_EXPERIMENTS
    if (threadIdx.x == 0) {
        GEMM_MARK(7);
        if (args.trace && blockIdx.x < 2) {
            const unsigned long long t0 = wend_s[0];
            double e[12];
            for (int w = 0; w < 12; ++w) e[w] = (double)(long long)(wend_s[w] - t0) * 1e-3;
            printf("k_gemmq<%d> cta%d warp ends rel. to warp 0 (us): %.2f %.2f %.2f %.2f %.2f %.2f %.2f %.2f %.2f "
                   "%.2f %.2f %.2f\n", kMode, (int)blockIdx.x, e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7], e[8],
                   e[9], e[10], e[11]);
        }
        if (args.trace && blockIdx.x == 0) {
            const unsigned long long* m = tmark_s;
            printf("k_gemmq<%d> cta0 (us): setup %.2f | griddep %.2f | first operands %.2f | last commit %.2f | "
                   "first drain %.2f | drained %.2f | row scale %.2f | epilogue end %.2f | teardown %.2f\n", kMode,
                   (m[1] - m[0]) * 1e-3, (m[2] - m[1]) * 1e-3, (m[3] - m[2]) * 1e-3, (m[4] - m[0]) * 1e-3,
                   (m[5] - m[0]) * 1e-3, (m[8] - m[0]) * 1e-3, (m[9] - m[0]) * 1e-3, (m[6] - m[0]) * 1e-3,
                   (m[7] - m[6]) * 1e-3);
        }
    }
#endif
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

// Q-layout viewed as a 3-D byte array [slice][(kb * rows_total + row) / 4][256]:
// four consecutive 64-byte Q-rows form one 256-byte TMA row (the data is
// pre-swizzled, SWIZZLE_NONE copies bytes), so a stage of box_rows Q-rows x 3
// slices is fetched as 3 * box_rows / 4 wide requests instead of 3 * box_rows
// 64-byte ones -- the TMA request rate, not bandwidth, limited the 64-byte form.
bool make_q_tmap(void* map_out, const uint8_t* base, int64_t rows_total, int64_t nkb, int box_rows) {
    CUtensorMap* map = reinterpret_cast<CUtensorMap*>(map_out);
    auto fn = encode_fn();
    if (!fn) return false;
    if ((rows_total * nkb) % 4 || box_rows % 4) return false;
    cuuint64_t dims[3] = {256, (cuuint64_t)(rows_total * nkb / 4), (cuuint64_t)kSlices};
    cuuint64_t strides[2] = {256, (cuuint64_t)(rows_total * nkb * 64)};
    cuuint32_t box[3] = {256, (cuuint32_t)(box_rows / 4), (cuuint32_t)kSlices};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

#ifdef SOS_EXPERIMENTS
// Experiment build only (-DSOS_EXPERIMENTS, never the shipped library): tuning
// and diagnostic switches read from the environment, see DESIGN.md 5.4.
static int env_int(const char* name, int dflt) {
    const char* s = getenv(name);
    return s && *s ? atoi(s) : dflt;
}
#endif

// CTAs of k_gemmq<kMode> that can be resident at once (2 per co-resident
// cluster): the bounded K-skew waits for all CTAs of the grid, so the grid
// must never exceed it (else every epoch would run into the spin bound)
template <int kMode>
static int resident_ctas(int num_sms) {
    static int cached = -1;
    if (cached < 0) {
        cudaFuncSetAttribute(k_gemmq<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(num_sms & ~1);
        cfg.blockDim = dim3(kGemmThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k_gemmq<kMode>, &cfg) != cudaSuccess || nc <= 0) {
            cudaGetLastError();
            nc = num_sms / 2;
        }
        cached = std::min(num_sms, 2 * nc);
    }
    return cached;
}

int resident_gemm_pairs(int num_sms) { return resident_ctas<kModeFwd>(num_sms) / 2; }

template <int kMode>
static cudaError_t launchq(const Plan& P, const CUtensorMap& ma, const CUtensorMap& mb, GemmArgs a,
                           cudaStream_t st, bool pdl = false) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_gemmq<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        configured = true;
    }
    int sms = resident_ctas<kMode>(P.num_sms);
    // bounded K-skew only when the operands do not fit in L2 anyway: for short K
    // (both operand tensors <= kSkewMinBytes) the pacing is a soft grid barrier
    // every kSkewEpoch K-blocks with nothing to gain (config 2: -5 % step time
    // without it, profiles/r2_short_k_ab.log)
    const bool pace = (double)(a.a_rows + a.b_rows) * a.num_kb * 64 * kSlices > kSkewMinBytes;
    a.skew_epoch = pace ? kSkewEpoch : 1 << 30;
    a.skew_lag = kSkewLag;
    a.skew_sleep = 256;
    a.kserp = 1;
#ifdef SOS_EXPERIMENTS
    {
        static const int epoch = env_int("SOS_SKEW_EPOCH", kSkewEpoch), lag = env_int("SOS_SKEW_LAG", kSkewLag);
        a.skew_epoch = epoch > 0 ? epoch : 1 << 30;
        a.skew_lag = lag;
        a.skew_sleep = env_int("SOS_SKEW_SLEEP", 256);
        a.probe = env_int("SOS_GEMM_PROBE", 0);
        a.skip_red = env_int("SOS_FWD_SKIP", 0);
        a.kserp = env_int("SOS_KSERP", 1);
        static unsigned long long* dbg = nullptr;
        if (env_int("SOS_GEMM_STATS", 0)) {
            if (!dbg && cudaMalloc(&dbg, 8 * sizeof(unsigned long long)) == cudaSuccess)
                cudaMemset(dbg, 0, 8 * sizeof(unsigned long long));
            a.dbg = dbg;
        }
        a.trace = env_int("SOS_GEMM_TRACE", 0);
        const int max_ctas = env_int("SOS_GEMM_CTAS", 0);  // cap the persistent grid
        if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;
    }
#endif
    int grid = 2 * a.ntiles < sms ? 2 * a.ntiles : sms;
    grid &= ~1;
    if (grid <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_gemmq<kMode>, ma, mb, a);
#ifdef SOS_EXPERIMENTS
    if (a.dbg) {  // SOS_GEMM_STATS: wait cycles summed over CTAs, per launch (instrumentation only)
        unsigned long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost);
        cudaMemset(a.dbg, 0, sizeof(h));
        const double mma_total = (double)h[4];
        fprintf(stderr,
                "gemm_stats mode=%d grid=%d | per leader CTA (Mcycles): mma_thread_total=%.2f full_wait=%.2f (%.1f%%) "
                "tempty_wait=%.2f (%.1f%%) | per CTA producer: skew_wait=%.2f empty_wait=%.2f\n",
                kMode, grid, mma_total / (grid / 2) / 1e6, (double)h[3] / (grid / 2) / 1e6, 100.0 * h[3] / mma_total,
                (double)h[2] / (grid / 2) / 1e6, 100.0 * h[2] / mma_total, (double)h[0] / grid / 1e6,
                (double)h[1] / grid / 1e6);
    }
#endif
    return e;
}

static const CUtensorMap& tm(const uint8_t* raw) { return *reinterpret_cast<const CUtensorMap*>(raw); }

// The V^T slices for the backward come from the forward's two aux warps when
// the forward is long enough to hide them (elements per aux thread vs K-blocks
// per CTA pair, over the grid the forward actually launches: ~2.5 elements fit
// under one K-block's MMAs), else from the all-SM k_pack_vtq before the GEMM
// (small / mid-size problems).
bool vtq_fits_aux(const Plan& P) {
    const int grid = std::min<int64_t>(2 * (int64_t)P.ntiles_fwd, P.num_sms) & ~1;
    if (grid <= 0) return false;
    const double pairs = grid / 2, aux_threads = grid * 64.0;
    const double elems_per_thread = (double)P.idx->N * P.r / aux_threads;
    const double kblocks_per_pair = std::ceil(P.ntiles_fwd / pairs) * P.nkbV;
    return elems_per_thread <= 2.5 * kblocks_per_pair;
}

void launch_gemm_fwd(Plan& P, float* coef, const float* V_for_vtq, cudaStream_t st, const unsigned* urow,
                     const unsigned* vcol, bool zero_scal, bool pdl) {
    if (V_for_vtq && !P.vtq_in_aux) {
        launch_pack_vtq(P, V_for_vtq, st, vcol);
        V_for_vtq = nullptr;
    }
    GemmArgs a{};
    a.Vsrc = V_for_vtq;
    a.vtq = P.d_vtq;
    a.rowsVT = P.rowsVT;
    a.nkbN = P.nkbN;
    a.vcol = vcol ? vcol : P.d_vcol;
    a.r = P.r;
    a.a_rows = P.rowsV;
    a.b_rows = P.rowsV;
    a.num_kb = (int)P.nkbV;
    a.seg_kb = kSegKBMax;
    a.tiles = P.d_tiles_fwd;
    a.ntiles = P.ntiles_fwd;
    a.umaxA = urow ? urow : P.d_vrow;
    a.umaxB = a.umaxA;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.pt = P.idx->d_pt;
    a.coef = coef;
    a.zero_scal = zero_scal ? P.d_scal : nullptr;
    a.progress = P.d_progress;
    LaunchScope ls(P, KK_GEMM_FWD, st);
    launchq<kModeFwd>(P, tm(P.tmap_vq_a), tm(P.tmap_vq_b), a, st, pdl && !ls.a);
}

static GemmArgs bwd_args(Plan& P, const unsigned* vcol) {
    GemmArgs a{};
    a.a_rows = P.idx->Np;
    a.b_rows = P.rowsVT;
    a.num_kb = (int)P.nkbN;
    a.seg_kb = kSegKBMax;
    a.tiles = P.d_tiles_bwd;
    a.ntiles = P.ntiles_bwd;
    a.umaxA = P.d_rrow;
    a.umaxB = vcol ? vcol : P.d_vcol;
    a.N = P.idx->N;
    a.Np = P.idx->Np;
    a.r = P.r;
    a.scal = P.d_scal;
    a.progress = P.d_progress + 1;
    return a;
}

void launch_gemm_bwd(Plan& P, float* grad, cudaStream_t st, const unsigned* vcol, const uint8_t* tmap_vtq, bool pdl) {
    GemmArgs a = bwd_args(P, vcol);
    a.grad = grad;
    LaunchScope ls(P, KK_GEMM_BWD, st);
    launchq<kModeBwdStore>(P, tm(P.tmap_rq_a), tm(tmap_vtq ? tmap_vtq : P.tmap_vtq_b), a, st, pdl && !ls.a);
}

// backward whose finished gradient tiles are consumed in the same kernel by the
// optimiser step (GD or Adam): the gradient never makes an HBM round trip.  The
// GEMM reads the packed copy VTQ, never V, so updating V in place is safe.
void launch_gemm_bwd_update(Plan& P, float* V, cudaStream_t st, const DescendBufs* db) {
    GemmArgs a = bwd_args(P, db ? db->ucol_cur : nullptr);
    if (db && db->urow_r) a.umaxA = db->urow_r;
    if (db) {
        a.vq_next = P.d_vq;
        a.rowsV = P.rowsV;
        a.nkbV = P.nkbV;
        a.vrow_cur = db->vrow_cur;
        a.vrow_next = db->vrow_next;
        a.vcol_next = db->vcol_next;
        // the next step's V^T slices (scale kHeadroom x the current column maximum)
        a.vtq = db->vtq_next;
        a.vcol = db->vcol_cur;
        a.rowsVT = P.rowsVT;
        a.nkbN = P.nkbN;
    }
    a.ring = P.d_ring;
    a.V = V;
    a.opt = P.d_opt;
    a.use_stop = 1;
    a.adam = P.opt_kind == 1;
    if (a.adam) {
        a.m = P.d_m;
        a.v = P.d_v;
    }
    if (P.sig_on) {
        a.rowsig = P.d_rowsig;
        a.sig_blocks = P.sig_blocks;
        a.sig_chunks = (int)P.sig_expect.size();
    }
    LaunchScope ls(P, KK_GEMM_BWD, st);
    if (a.vtq)
        launchq<kModeBwdUpdateVtq>(P, tm(P.tmap_rq_a), tm(db->tmap_vtq_cur), a, st);
    else
        launchq<kModeBwdUpdate>(P, tm(P.tmap_rq_a), tm(db ? db->tmap_vtq_cur : P.tmap_vtq_b), a, st);
}

}  // namespace sos

// sos_pointwise.cu -- HBM-bound kernels of the step: per-row maxima and int8
// slice packing of V, V^T and of the residual matrix R (R_ij = res[rank(alpha_i +
// alpha_j)], gathered through the pair-rank table), and the fused residual +
// loss reduction.  The optimiser update of PAPER.md:221 runs inside the backward
// GEMM (sos_gemmq.cu).  All kernels are coalesced and sized as a multiple of
// the SM count (grid-stride).
#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sm100_ptx.cuh"
#include "sos_internal.cuh"
#include "sos_slice.cuh"

namespace sos {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------- V maxima ----
// vrow[i] = max_k |V_ik|, vcol[k] = max_i |V_ik| in one read of V (float bits,
// atomicMax on non-negative floats).  Block tile: 64 rows x 1024 columns,
// thread = 4 consecutive columns (float4), 8 rows in flight per thread; row
// maxima are warp-reduced per row and combined across the 8 warps in shared
// memory, so a tile issues 64 + 1024 atomics.
__global__ void __launch_bounds__(256) k_vmax(const float* __restrict__ V, int64_t N, int64_t r,
                                              unsigned* __restrict__ vrow, unsigned* __restrict__ vcol) {
    __shared__ float rowred[64][8];
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int64_t ntr = (N + 63) / 64, ntc = (r + 1023) / 1024;
    const bool vec = (r & 3) == 0;
    for (int64_t tile = blockIdx.x; tile < ntr * ntc; tile += gridDim.x) {
        const int64_t i0 = (tile / ntc) * 64, k0 = (tile % ntc) * 1024 + 4 * t;
        float cm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (int rr0 = 0; rr0 < 64; rr0 += 8) {
            float4 x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int64_t i = i0 + rr0 + e;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < N) {
                    if (vec && k0 + 4 <= r) {
                        v = __ldg(reinterpret_cast<const float4*>(V + i * r + k0));
                    } else {
                        if (k0 < r) v.x = __ldg(V + i * r + k0);
                        if (k0 + 1 < r) v.y = __ldg(V + i * r + k0 + 1);
                        if (k0 + 2 < r) v.z = __ldg(V + i * r + k0 + 2);
                        if (k0 + 3 < r) v.w = __ldg(V + i * r + k0 + 3);
                    }
                }
                x[e] = v;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float a0 = fabsf(x[e].x), a1 = fabsf(x[e].y), a2 = fabsf(x[e].z), a3 = fabsf(x[e].w);
                cm[0] = fmaxf(cm[0], a0);
                cm[1] = fmaxf(cm[1], a1);
                cm[2] = fmaxf(cm[2], a2);
                cm[3] = fmaxf(cm[3], a3);
                const float m = warp_max(fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
                if (lane == 0) rowred[rr0 + e][w] = m;
            }
        }
        __syncthreads();
        if (t < 64) {
            float m = rowred[t][0];
#pragma unroll
            for (int q = 1; q < 8; ++q) m = fmaxf(m, rowred[t][q]);
            if (i0 + t < N && m > 0.f) atomicMax(vrow + i0 + t, __float_as_uint(m));
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (k0 + e < r && cm[e] > 0.f) atomicMax(vcol + k0 + e, __float_as_uint(cm[e]));
        __syncthreads();
    }
}

// --------------------------------------------------------------- pack VQ ----
// thread = (row i, 16-wide K chunk): one 64-byte read (float4 when r % 4 == 0),
// 4 consecutive threads fill one 64-byte Q-row of each slice.  Rows >= N and
// K >= r are written as zeros.
__global__ void __launch_bounds__(256, 6) k_pack_vq(const float* __restrict__ V, int64_t N, int64_t r, int64_t rowsV,
                                                 int64_t nkb, const unsigned* __restrict__ vrow,
                                                 uint8_t* __restrict__ VQ) {
    const int64_t cpr = nkb * 4;  // chunks per row
    const int64_t total = rowsV * cpr;
    const bool vec = (r & 3) == 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / cpr, cc = t - i * cpr;
        const int64_t k0 = cc * 16;
        float x[16];
        float c = 0.f;
        if (i < N) {
            c = slice_scale(__ldg(vrow + i));
            if (vec && k0 + 16 <= r) {
                const float4* s = reinterpret_cast<const float4*>(V + i * r + k0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 f = __ldg(s + q);
                    x[4 * q] = f.x; x[4 * q + 1] = f.y; x[4 * q + 2] = f.z; x[4 * q + 3] = f.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) x[e] = k0 + e < r ? __ldg(V + i * r + k0 + e) : 0.f;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = 0.f;
        }
        uint4 q[3];
        slice16(x, c, q);
        store_q16(VQ, cc >> 2, i, (int)(cc & 3), nkb, rowsV, q);
    }
}

// -------------------------------------------------------------- pack VTQ ----
// (tile routine pack_vtq_tile in sos_slice.cuh, shared with the forward GEMM's aux warps)
__global__ void __launch_bounds__(256) k_pack_vtq(const float* __restrict__ V, int64_t N, int64_t r,
                                                  int64_t rowsVT, int64_t nkbN, const unsigned* __restrict__ vcol,
                                                  uint8_t* __restrict__ VTQ) {
    __shared__ float tile[64][65];
    const int64_t nkt = (rowsVT + 63) / 64;
    for (int64_t b = blockIdx.x; b < nkbN * nkt; b += gridDim.x)
        pack_vtq_tile<256>(V, N, r, rowsVT, nkbN, vcol, VTQ, b / nkt, (b % nkt) * 64, tile, threadIdx.x);
}

// ------------------------------------------------------------- residual ----
// res = coef - p ; loss += res^2 ; pnorm2 += p^2
__global__ void k_residual(const float* __restrict__ coef, const float* __restrict__ p, float* __restrict__ res,
                           int64_t M, Scalars* __restrict__ sc) {
    double l = 0.0, pn = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += stride) {
        const float pv = p[t];
        const float rv = coef[t] - pv;
        res[t] = rv;
        l += (double)rv * rv;
        pn += (double)pv * pv;
    }
    l = warp_sum(l);
    pn = warp_sum(pn);
    __shared__ double s_l[32], s_p[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_l[w] = l; s_p[w] = pn; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        l = lane < nw ? s_l[lane] : 0.0;
        pn = lane < nw ? s_p[lane] : 0.0;
        l = warp_sum(l);
        pn = warp_sum(pn);
        if (lane == 0) {
            atomicAdd(&sc->loss, l);
            atomicAdd(&sc->pnorm2, pn);
        }
    }
}

// ---------------------------------------------------------------- R maxima --
// rrow[i] = max_j |res[rank(alpha_i + alpha_j)]| by one pass over the stored
// block triangle of PT: a CTA gathers one 64 x 64 block {I <= J} of |R| into
// shared memory and folds it into the maxima of the rows of I (across the
// block's columns) and of the rows of J (across its rows: R is symmetric) with
// atomicMax on float bits (rrow zeroed before).  Used when N^2 lookups are
// cheaper than the lattice DP (small problems, many variables).
__global__ void __launch_bounds__(256) k_rmax(const uint32_t* __restrict__ pt, const float* __restrict__ res,
                                              int64_t nkb, unsigned* __restrict__ rrow, const Scalars* sc,
                                              const DevOpt* opt, int use_stop) {
    if (descent_stopped(sc, opt, use_stop)) return;
    __shared__ __align__(16) float tile[kPtW * kPtW];  // slots swizzled (rt_slot)
    const int t = threadIdx.x;
    const int64_t npairs = nkb * (nkb + 1) / 2;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
        int64_t J = (int64_t)((sqrt(8.0 * (double)pr + 1.0) - 1.0) * 0.5);
        while (J * (J + 1) / 2 > pr) --J;
        while ((J + 1) * (J + 2) / 2 <= pr) ++J;
        const int64_t I = pr - J * (J + 1) / 2;
        const uint32_t* p0 = pt + pt_entry(I * kPtW, J * kPtW);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int row, col4;
            rt_gather_pos(t, u, row, col4);
            const uint4 k = __ldg(reinterpret_cast<const uint4*>(p0 + row * 64 + col4 * 4));
            rt_store4<kGatherBlocks>(tile, row, col4,
                      make_float4(k.x != kInvalidRank ? fabsf(__ldg(res + k.x)) : 0.f,
                                  k.y != kInvalidRank ? fabsf(__ldg(res + k.y)) : 0.f,
                                  k.z != kInvalidRank ? fabsf(__ldg(res + k.z)) : 0.f,
                                  k.w != kInvalidRank ? fabsf(__ldg(res + k.w)) : 0.f));
        }
        __syncthreads();
        // thread t: row (t >> 2) of I across columns 16 (t & 3) .. +15, and column
        // (t >> 2) of the block = row of J across rows 16 (t & 3) .. +15
        const int line = t >> 2, part = t & 3;
        float x[16];
        rt_row16<kGatherBlocks>(tile, line, part, x);
        float mr = 0.f, mc = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            mr = fmaxf(mr, x[e]);                               // row `line` of I
            mc = fmaxf(mc, rt_at<kGatherBlocks>(tile, part * 16 + e, line));   // column `line` = row of J
        }
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 1));
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 2));
        mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 1));
        mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 2));
        if (part == 0) {
            if (mr > 0.f) atomicMax(rrow + I * kPtW + line, __float_as_uint(mr));
            if (I != J && mc > 0.f) atomicMax(rrow + J * kPtW + line, __float_as_uint(mc));
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------- pack RQ ----
// R is symmetric (R_ij = res[rank(alpha_i + alpha_j)] = R_ji): one 64 x 64 block of
// PT is read per unordered block pair {I <= J} and both RQ blocks -- rows of I at
// K-block J and rows of J at K-block I (the transposed tile) -- are written from
// it, so PT and the res gathers are read once for two blocks.  RQ rows at or
// beyond nkb * 64 (padding of Np) are never written: zeroed at plan creation.
// kHr (inside sos_descend after its first step): the row scales are not known
// yet -- the slices use kHeadroom x the previous step's exact row maximum
// (rrow_prev), and the exact maxima of this step's R rows are folded into
// rrow_out (atomicMax, cleared by k_step_begin) from the tiles already in shared
// memory; k_rfix then re-slices the rare rows whose maximum left [u/4, u].
// This takes the lattice DP (0.32 ms at config 4) off the step.
template <bool kHr>
__global__ void __launch_bounds__(256, 6) k_pack_rq_sym(const uint32_t* __restrict__ pt, const float* __restrict__ res,
                                                     int64_t Np, int64_t nkb, const unsigned* __restrict__ rrow,
                                                     uint8_t* __restrict__ RQ, const Scalars* sc, const DevOpt* opt,
                                                     int use_stop, unsigned* __restrict__ rrow_out) {
    if (descent_stopped(sc, opt, use_stop)) return;
    __shared__ __align__(16) float tile[kPtW * kPtW];  // [row in I][j in J], slots swizzled (rt_slot)
    const int t = threadIdx.x;
    const int64_t npairs = nkb * (nkb + 1) / 2;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
        // pr enumerates the upper triangle column by column: J, then I = 0..J
        int64_t J = (int64_t)((sqrt(8.0 * (double)pr + 1.0) - 1.0) * 0.5);
        while (J * (J + 1) / 2 > pr) --J;
        while ((J + 1) * (J + 2) / 2 <= pr) ++J;
        const int64_t I = pr - J * (J + 1) / 2;
        const uint32_t* p0 = pt + pt_entry(I * kPtW, J * kPtW);  // 64 rows x 64 ranks, contiguous
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int row, col4;
            rt_gather_pos(t, u, row, col4);
            const uint4 k = __ldg(reinterpret_cast<const uint4*>(p0 + row * 64 + col4 * 4));
            rt_store4<kGatherBlocks>(tile, row, col4,
                      make_float4(k.x != kInvalidRank ? __ldg(res + k.x) : 0.f, k.y != kInvalidRank ? __ldg(res + k.y) : 0.f,
                                  k.z != kInvalidRank ? __ldg(res + k.z) : 0.f, k.w != kInvalidRank ? __ldg(res + k.w) : 0.f));
        }
        __syncthreads();
        const int r = t >> 2, c = t & 3;
        float x[16];
        uint4 q[3];
        float mr = 0.f;
        rt_row16<kGatherBlocks>(tile, r, c, x);
        if (kHr) {
#pragma unroll
            for (int e = 0; e < 16; ++e) mr = fmaxf(mr, fabsf(x[e]));
        }
        const unsigned urI = kHr ? __float_as_uint(kHeadroom * __uint_as_float(__ldg(rrow + I * kPtW + r)))
                                 : __ldg(rrow + I * kPtW + r);
        slice16(x, slice_scale(urI), q);
        store_q16(RQ, J, I * kPtW + r, c, nkb, Np, q);
        float mc = 0.f;
        if (I != J) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                x[e] = rt_at<kGatherBlocks>(tile, c * 16 + e, r);
                if (kHr) mc = fmaxf(mc, fabsf(x[e]));
            }
            const unsigned urJ = kHr ? __float_as_uint(kHeadroom * __uint_as_float(__ldg(rrow + J * kPtW + r)))
                                     : __ldg(rrow + J * kPtW + r);
            slice16(x, slice_scale(urJ), q);
            store_q16(RQ, I, J * kPtW + r, c, nkb, Np, q);
        }
        if (kHr) {  // exact maxima: rows of I over J's columns, rows of J over I's (4 threads per line)
            mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 1));
            mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 2));
            mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 1));
            mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 2));
            if (c == 0) {
                if (mr > 0.f) atomicMax(rrow_out + I * kPtW + r, __float_as_uint(mr));
                if (I != J && mc > 0.f) atomicMax(rrow_out + J * kPtW + r, __float_as_uint(mc));
            }
        }
        __syncthreads();
    }
}

// After k_pack_rq_sym<true>: row i's slices used u = kHeadroom * (previous
// exact maximum); they are exact to ~22 bits while the new exact maximum lies
// in [u/4, u] (the same window as V's, k_descend_fixup).  Outside it -- growth
// beyond the headroom would overflow the top slice, a large shrink loses bits,
// and the first step after a zero row -- one warp re-gathers row i through PT
// and re-slices it with the exact maximum.  urow_r receives the scale each RQ
// row was written with (the backward's A unscale).  A stopped descent carries
// the previous maxima over (no backward runs).
__global__ void __launch_bounds__(256) k_rfix(const uint32_t* __restrict__ pt, const float* __restrict__ res,
                                              int64_t N, int64_t Np, int64_t nkb, const unsigned* __restrict__ rrow_prev,
                                              unsigned* __restrict__ rrow_cur, unsigned* __restrict__ urow_r,
                                              uint8_t* __restrict__ RQ, const Scalars* sc, const DevOpt* opt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (descent_stopped(sc, opt, 1)) {
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < Np; e += (int64_t)gridDim.x * blockDim.x)
            rrow_cur[e] = rrow_prev[e];
        return;
    }
    for (int64_t i = warp; i < N; i += nwarps) {
        const float u = kHeadroom * __uint_as_float(rrow_prev[i]);
        const unsigned mb = rrow_cur[i];
        const float mx = __uint_as_float(mb);
        const bool keep = mx <= u && mx >= 0.25f * u;
        if (lane == 0) urow_r[i] = keep ? __float_as_uint(u) : mb;
        if (keep) continue;
        const float cs = slice_scale(mb);
        for (int64_t cc = lane; cc < nkb * 4; cc += 32) {  // 16-column chunks of row i
            const int64_t j0 = cc * 16;
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int64_t j = j0 + e;
                const uint32_t k = j < N ? pt[pt_entry_sym(i, j)] : kInvalidRank;
                x[e] = k != kInvalidRank ? res[k] : 0.f;
            }
            uint4 q[3];
            slice16(x, cs, q);
            store_q16(RQ, cc >> 2, i, (int)(cc & 3), nkb, Np, q);
        }
    }
}

// -------------------------------------------------------------- launches ---
// blocks of `fn` that fit on one SM at once (occupancy API, cached per kernel)
static int resident_per_sm(const void* fn, int threads, size_t smem) {
    struct Entry { const void* fn; int threads; size_t smem; int nb; };
    static std::vector<Entry> cache;
    static std::mutex mu;  // distinct plans may launch from distinct host threads
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
        if (e.fn == fn && e.threads == threads && e.smem == smem) return e.nb;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    cache.push_back(Entry{fn, threads, smem, nb});
    return nb;
}
// grid of a grid-stride kernel: enough blocks for the work, but never more than
// fit on the GPU at once (more would run a partial second wave with the same
// per-block work: the R packer at config 4 ran 1184 blocks on 888 slots)
template <typename F>
static int grid_for(const Plan& P, F* fn, int64_t work, int threads, int per_sm = 64, size_t smem = 0) {
    int64_t b = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)P.num_sms * std::min(per_sm, resident_per_sm((const void*)fn, threads, smem));
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

void launch_vmax(Plan& P, const float* V, cudaStream_t st, unsigned* vrow, unsigned* vcol) {
    const int64_t N = P.idx->N;
    if (!vrow) vrow = P.d_vrow;
    if (!vcol) vcol = P.d_vcol;
    cudaMemsetAsync(vrow, 0, P.rowsV * sizeof(unsigned), st);
    cudaMemsetAsync(vcol, 0, P.rowsVT * sizeof(unsigned), st);
    LaunchScope ls(P, KK_ABSMAX_V, st);
    const int64_t tiles = ((N + 63) / 64) * ((P.r + 1023) / 1024);
    k_vmax<<<grid_for(P, k_vmax, tiles * 256, 256), 256, 0, st>>>(V, N, P.r, vrow, vcol);
}

void launch_pack_vtq(Plan& P, const float* V, cudaStream_t st, const unsigned* vcol) {
    LaunchScope ls(P, KK_PACK_V, st);
    const int64_t blocks = P.nkbN * ((P.rowsVT + 63) / 64);
    k_pack_vtq<<<grid_for(P, k_pack_vtq, blocks * 256, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.rowsVT, P.nkbN,
                                                               vcol ? vcol : P.d_vcol, P.d_vtq);
}

void launch_residual(Plan& P, const float* coef, const float* p, float* res, cudaStream_t st) {
    LaunchScope ls(P, KK_RESIDUAL, st);
    k_residual<<<grid_for(P, k_residual, P.idx->M, 256, 4), 256, 0, st>>>(coef, p, res, P.idx->M, P.d_scal);
}

// rrow_zeroed: the caller cleared rrow in the same stream (k_step_begin inside
// sos_descend, so the replayed steps hold no memset node)
void launch_rmax(Plan& P, const float* res, cudaStream_t st, int use_stop, bool rrow_zeroed) {
    LaunchScope ls(P, KK_ABSMAX_R, st);
    if (!rrow_zeroed) cudaMemsetAsync(P.d_rrow, 0, (size_t)P.idx->Np * sizeof(unsigned), st);
    const int64_t nkb = P.idx->Np / kPtW, npairs = nkb * (nkb + 1) / 2;
    const unsigned blocks = grid_for(P, k_rmax, npairs * 256, 256);
    k_rmax<<<blocks, 256, 0, st>>>(P.idx->d_pt, res, nkb, P.d_rrow, P.d_scal, P.d_opt, use_stop);
}

// step bookkeeping (one thread: Adam t += 1; inside sos_descend the loss of
// this step into the call's array) and zeroing of accumulators: the next
// step's maxima (zero0 / zero1: n0 / n1 words), the R row maxima of the direct
// pass (zero2: n2 words) and the coefficient accumulator of the next forward
// (zc: nc floats, 16-B aligned)
__global__ void k_step_begin(DevOpt* opt, const Scalars* sc, double* losses, int from_opt, unsigned* zero0,
                             int64_t n0, unsigned* zero1, int64_t n1, unsigned* zero2, int64_t n2, float* zc,
                             int64_t nc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        advance_step(opt);
        if (from_opt) losses = opt->losses;
        if (losses) losses[opt->loss_idx++] = sc->loss;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t e = tid; e < n0 + n1 + n2; e += stride) {
        if (e < n0) zero0[e] = 0u;
        else if (e < n0 + n1) zero1[e - n0] = 0u;
        else zero2[e - n0 - n1] = 0u;
    }
    for (int64_t e = tid; e < nc / 4; e += stride) reinterpret_cast<float4*>(zc)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = (nc / 4) * 4 + tid; e < nc; e += stride) zc[e] = 0.f;
}

// ------------------------------------------------- split step: update ----
// GD / Adam on a block of `rows` (1, 2 or 4) whole rows of V, in
// two passes.  Pass 1 is purely elementwise: the block's rows are one contiguous
// span of V, m, v and the gradient (16-byte aligned: rows * r is a multiple of
// 4), streamed as float4 with kUpdU of them in flight per array and
// thread; the new values also go to a shared-memory copy of the span (or, for
// rows longer than kUpdSmemR, are re-read from L2).  Pass 2 takes the EXACT
// maximum of each new row (one warp per row) and slices the rows into the next
// step's VQ against it (thread = 4 K-values, one word per slice): no headroom
// scale, no fixup kernel.  (The column maxima of V_{t+1}, for its V^T slices,
// are taken by the next k_mid.)  A stopped descent (sos_opt_set_stop) leaves V,
// m, v and VQ unchanged and carries the row maxima over.
constexpr int kUpdRows = 4, kUpdThreads = 256, kUpdU = 2;  // kUpdRows: the most rows per block
constexpr int64_t kUpdSmemR = 4096;  // rows up to this length are staged in shared memory (64 KB)
__device__ __forceinline__ float adam_or_gd(bool adam, float x, float g, float& m, float& v, const DevOpt& o) {
    if (!adam) return x - o.lr * g;
    m = o.b1 * m + (1.f - o.b1) * g;
    v = o.b2 * v + (1.f - o.b2) * g * g;
    return x - o.lr_c1 * m / (sqrtf(v) * o.inv_sqrt_c2 + o.eps);
}
__global__ void __launch_bounds__(kUpdThreads) k_update_rows(
    const float* __restrict__ grad, float* V, float* __restrict__ m, float* __restrict__ v, int64_t N, int64_t r,
    int adam, const DevOpt* opt, const Scalars* sc, uint8_t* __restrict__ vq_next, int64_t rowsV, int64_t nkbV,
    const unsigned* __restrict__ vrow_cur, unsigned* __restrict__ vrow_next, int keep_l2, int rows) {
    extern __shared__ float4 stage4[];  // the block's span (flat), when r <= kUpdSmemR
    __shared__ float rmax_s[kUpdRows];
    griddep_wait();  // launched with programmatic stream serialization after the backward
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * rows;
    const int nr = (int)(N - i0 < rows ? N - i0 : rows);
    if (descent_stopped(sc, opt, 1)) {
        if (vrow_next && t < nr) vrow_next[i0 + t] = vrow_cur[i0 + t];
        return;
    }
    const DevOpt o = *opt;
    // evict_last keeps V, m, v in L2 from step to step when they fit in it (keep_l2:
    // config 2 +1.9 %, N = 2926 +2.8 %, profiles/r2_short_k_ab.log), else evict_first
    const uint64_t pol = keep_l2 ? l2_evict_last_policy() : l2_evict_first_policy();
    const bool in_smem = r <= kUpdSmemR;
    const int64_t base = i0 * r, len = nr * r, n4 = len >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(grad + base);
    float4* V4 = reinterpret_cast<float4*>(V + base);
    float4* m4 = reinterpret_cast<float4*>(m + base);
    float4* v4 = reinterpret_cast<float4*>(v + base);
    for (int64_t q0 = t; q0 < n4; q0 += kUpdThreads * kUpdU) {
        float4 gv[kUpdU], x[kUpdU], mm[kUpdU], vv[kUpdU];
#pragma unroll
        for (int u = 0; u < kUpdU; ++u) {
            const int64_t q = q0 + kUpdThreads * u;
            if (q < n4) {
                gv[u] = __ldcs(g4 + q);
                x[u] = ld_f4_hint(V4 + q, pol);
                if (adam) {
                    mm[u] = ld_f4_hint(m4 + q, pol);
                    vv[u] = ld_f4_hint(v4 + q, pol);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUpdU; ++u) {
            const int64_t q = q0 + kUpdThreads * u;
            if (q >= n4) break;
            float4 xn;
            if (adam) {
                xn.x = adam_or_gd(true, x[u].x, gv[u].x, mm[u].x, vv[u].x, o);
                xn.y = adam_or_gd(true, x[u].y, gv[u].y, mm[u].y, vv[u].y, o);
                xn.z = adam_or_gd(true, x[u].z, gv[u].z, mm[u].z, vv[u].z, o);
                xn.w = adam_or_gd(true, x[u].w, gv[u].w, mm[u].w, vv[u].w, o);
                st_f4_hint(m4 + q, mm[u], pol);
                st_f4_hint(v4 + q, vv[u], pol);
            } else {
                xn = make_float4(x[u].x - o.lr * gv[u].x, x[u].y - o.lr * gv[u].y, x[u].z - o.lr * gv[u].z,
                                 x[u].w - o.lr * gv[u].w);
            }
            if (keep_l2) st_f4_hint(V4 + q, xn, pol);  // read again by the next k_mid
            else V4[q] = xn;
            if (in_smem) stage4[q] = xn;
        }
    }
    float* stage = reinterpret_cast<float*>(stage4);
    for (int64_t e = 4 * n4 + t; e < len; e += kUpdThreads) {  // ragged end of the last block's span
        float mm1 = adam ? m[base + e] : 0.f, vv1 = adam ? v[base + e] : 0.f;
        const float xn = adam_or_gd(adam, V[base + e], grad[base + e], mm1, vv1, o);
        V[base + e] = xn;
        if (adam) {
            m[base + e] = mm1;
            v[base + e] = vv1;
        }
        if (in_smem) stage[e] = xn;
    }
    __syncthreads();  // the new rows are in shared memory / in V (visible to the block)
    const float* src = in_smem ? stage : V + base;
    if (w < nr) {
        float mx = 0.f;
        for (int64_t c = lane; c < r; c += 32) mx = fmaxf(mx, fabsf(src[w * r + c]));
        mx = warp_max(mx);
        if (lane == 0) {
            rmax_s[w] = mx;
            if (vrow_next) vrow_next[i0 + w] = __float_as_uint(mx);
        }
    }
    if (!vq_next) return;
    __syncthreads();
    const int64_t nq = nkbV * 16;  // 4-value quads per VQ row (K padded to 64)
    for (int rr = 0; rr < nr; ++rr) {
        const float sc4 = slice_scale(__float_as_uint(rmax_s[rr]));
        const float* row = src + rr * r;
        for (int64_t qd = t; qd < nq; qd += kUpdThreads) {
            const int64_t k0 = 4 * qd;
            float xs[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) xs[e] = k0 + e < r ? row[k0 + e] : 0.f;
            uint32_t qw[3];
            slice4(xs, sc4, qw);
            const int64_t cq = qd >> 2;
#pragma unroll
            for (int sl = 0; sl < 3; ++sl)
                *reinterpret_cast<uint32_t*>(vq_next + q_offset(sl, cq >> 2, i0 + rr, (int)(cq & 3), nkbV, rowsV) +
                                             4 * (qd & 3)) = qw[sl];
        }
    }
}

void launch_update_rows(Plan& P, float* V, uint8_t* vq_next, const unsigned* vrow_cur, unsigned* vrow_next,
                        cudaStream_t st) {
    LaunchScope ls(P, KK_UPDATE, st);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_update_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kUpdRows * kUpdSmemR * 4));
        configured = true;
    }
    // rows per block: of 1, 2, 4 (rows * r a multiple of 4), the one whose last wave
    // is fullest (r = 4004: 4 rows = 64 KB per block ran 501 blocks on 444 slots,
    // 1.13 waves; 1 row, 2002 blocks on 592 slots); ties -> more rows
    const int64_t N = P.idx->N;
    int rows = P.upd_rows;
    double best = -1.0;
    for (int R = kUpdRows; R >= 1 && !P.upd_rows; R >>= 1) {
        if ((R * P.r) % 4) continue;
        const size_t sm = P.r <= kUpdSmemR ? (size_t)R * P.r * sizeof(float) : 0;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_update_rows, kUpdThreads, sm) != cudaSuccess || nb < 1) {
            cudaGetLastError();
            nb = 1;
        }
        const double blocks = (double)((N + R - 1) / R), slots = (double)P.num_sms * nb;
        const double eff = blocks / (std::ceil(blocks / slots) * slots);
        if (eff > best + 1e-9) {
            best = eff;
            rows = R;
        }
    }
    P.upd_rows = rows;  // once per plan
    const int64_t blocks = (N + rows - 1) / rows;
    const size_t smem = P.r <= kUpdSmemR ? (size_t)rows * P.r * sizeof(float) : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kUpdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = ls.a ? 0 : 1;
    cudaLaunchKernelEx(&cfg, k_update_rows, (const float*)P.d_grad, V, P.d_m, P.d_v, N, P.r, (int)(P.opt_kind == 1),
                       (const DevOpt*)P.d_opt, (const Scalars*)P.d_scal, vq_next, P.rowsV, P.nkbV, vrow_cur, vrow_next,
                       (double)N * P.r * 12 <= (double)P.l2_bytes ? 1 : 0, rows);
}

// --------------------------------------------------- split step: k_mid ----
// Everything between the forward and the backward of a split step in ONE
// cooperative kernel (three phases separated by grid barriers) instead of
// 5-7 dependent launches, which bound short-K steps:
//   A: res = coef - p, loss += res^2 and |p|^2 (fp64 block sums, the stopping
//      rule's inputs); with colmax, the column maxima of V (per 64 x 64 tile,
//      atomicMax into vcol, which the previous k_mid cleared); clear rrow and
//      the next step's column maxima (zero_cols)
//   B: t += 1 and the loss record; the V^T slices of V (exact column maxima);
//      unless stopped, each block gathers its 64 x 64 blocks {I <= J} of R
//      through PT into shared memory (they stay there) and folds them into the
//      row maxima of I and J (atomicMax); coef cleared for the next forward
//   C: unless stopped, the held R blocks are sliced into RQ (rows of I at
//      K-block J and, transposed, rows of J at K-block I) -- R is gathered
//      once, not once for the maxima and again for the slices
struct MidArgs {
    float* coef;
    const float* p;
    float* res;
    int64_t M;
    Scalars* sc;
    DevOpt* opt;
    double* losses;
    int losses_from_opt;
    const uint32_t* pt;
    int64_t Np, nkbN;
    unsigned* rrow;
    uint8_t* RQ;
    const float* V;
    int64_t N, r, rowsVT;
    unsigned* vcol;
    int colmax;
    uint8_t* VTQ;
    unsigned* zero_cols;
    double* part;  // [gridDim][2] per-block partial sums of the loss and |p|^2
    int hold;   // every block holds its R blocks from phase B to C (else C gathers them again)
    int r_slots;  // shared-memory tiles before the held V tiles (max(R blocks held, 1))
    int hold_v;   // V tiles every block holds from phase A to B (0: phase B reads V again)
    int trace;  // experiment build only
    unsigned long long* dbg;  // experiment build, trace: per-phase maxima over blocks
};

__device__ __forceinline__ void block_pair(int64_t pr, int64_t& I, int64_t& J) {
    // pr enumerates the upper block triangle column by column: J, then I = 0..J
    J = (int64_t)((sqrt(8.0 * (double)pr + 1.0) - 1.0) * 0.5);
    while (J * (J + 1) / 2 > pr) --J;
    while ((J + 1) * (J + 2) / 2 <= pr) ++J;
    I = pr - J * (J + 1) / 2;
}

constexpr int kMidThreads = 256;
constexpr size_t kMidTileBytes = (size_t)kPtW * (kPtW + 1) * sizeof(float);
constexpr int kMidMaxHeld = 12;  // R blocks a k_mid block can hold in shared memory (~200 KB)
constexpr int kMidMaxHeldV = 4;  // V tiles a k_mid block can hold from phase A to B

// the 64 x 64 block {I <= J} of R (I's rows x J's columns) gathered through the
// stored PT block into a swizzled shared-memory tile (rt_slot; the first 4096
// floats of a 64 x 65 slot; plain loads: res is written in the same kernel)
__device__ __forceinline__ void gather_r_tile(const uint32_t* __restrict__ pt, const float* res, int64_t I, int64_t J,
                                              float* tile, int t) {
    const uint32_t* p0 = pt + pt_entry(I * kPtW, J * kPtW);
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // row-major map: at config 2 (res ~370 KB) faster than rt_gather_pos
        const int e = (u * 256 + t) * 4;
        const uint4 k = __ldg(reinterpret_cast<const uint4*>(p0 + e));
        rt_store4<kGatherRows>(tile, e >> 6, (e & 63) >> 2,
                  make_float4(k.x != kInvalidRank ? res[k.x] : 0.f, k.y != kInvalidRank ? res[k.y] : 0.f,
                              k.z != kInvalidRank ? res[k.z] : 0.f, k.w != kInvalidRank ? res[k.w] : 0.f));
    }
}

#ifdef SOS_EXPERIMENTS
// SOS_MID_TRACE=1 (experiment build): block 0 prints the phase boundaries of k_mid
#define MID_MARK(k) do { if (a.trace && threadIdx.x == 0) { \
    unsigned long long now_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_)); tmark[k] = now_; } } while (0)
#else
#define MID_MARK(k) do { } while (0)
#endif

#ifdef SOS_EXPERIMENTS
// the trace code would raise the register count to 94 (2 blocks per SM): keep the
// release build's 4 blocks per SM so that traces describe the same grid
#define SOS_MID_BOUNDS __launch_bounds__(kMidThreads, 4)
#else
#define SOS_MID_BOUNDS __launch_bounds__(kMidThreads)
#endif
__global__ void SOS_MID_BOUNDS k_mid(const MidArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
#ifdef SOS_EXPERIMENTS
    unsigned long long tmark[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
    griddep_wait();  // launched with programmatic stream serialization after the forward
    MID_MARK(0);
    extern __shared__ float smem_tiles[];  // R blocks held from phase B to C, 64 x 65 floats each
    __shared__ double red[2][kMidThreads / 32];
    float(*tile0)[kPtW + 1] = reinterpret_cast<float(*)[kPtW + 1]>(smem_tiles);
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + t, gstride = (int64_t)gridDim.x * blockDim.x;
    __shared__ float cpart[2][4][64];  // column maxima of two held V tiles, per 16-row group
    const double tol = a.opt->stop_tol;  // constant during the kernel: loaded up front
    // the step's bookkeeping (t += 1, the Adam constants, the loss record) is done
    // by the last block, which has the least work, at its very end (step_record)
    // ---- A
    {
        // this block's PT blocks into L2 now (read after the barrier; PT does not
        // stay in L2 across the GEMMs of a step)
        if (t < 128) {
            const int64_t npairs = a.nkbN * (a.nkbN + 1) / 2;
            for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
                int64_t I, J;
                block_pair(pr, I, J);
                prefetch_l2(a.pt + pt_entry(I * kPtW, J * kPtW) + t * 32);
            }
        }
        double l = 0.0, pn = 0.0;
        for (int64_t e = gtid; e < a.M; e += gstride) {
            const float pv = a.p[e];
            const float rv = a.coef[e] - pv;
            a.res[e] = rv;
            l += (double)rv * rv;
            pn += (double)pv * pv;
        }
        l = warp_sum(l);
        pn = warp_sum(pn);
        if (lane == 0) { red[0][w] = l; red[1][w] = pn; }
        __syncthreads();
        if (w == 0) {
            l = lane < kMidThreads / 32 ? red[0][lane] : 0.0;
            pn = lane < kMidThreads / 32 ? red[1][lane] : 0.0;
            l = warp_sum(l);
            pn = warp_sum(pn);
            if (lane == 0) {  // per-block partial sums (fp64 atomics from every block serialise)
                a.part[2 * blockIdx.x] = l;
                a.part[2 * blockIdx.x + 1] = pn;
            }
        }
        MID_MARK(9);
        for (int64_t e = gtid; e < a.Np; e += gstride) a.rrow[e] = 0u;
        if (a.zero_cols)
            for (int64_t e = gtid; e < a.rowsVT; e += gstride) a.zero_cols[e] = 0u;
        if (a.hold_v) {
            // this block's V tiles (64 rows j x 64 columns k of V; tile b = jb * nkt + kt,
            // b = blockIdx.x + h * gridDim.x) are read once, here, into shared memory and
            // sliced from there in phase B; two tiles' loads are in flight together and
            // the column maxima come from the registers (thread = column t & 63 of rows
            // (t >> 6) + 4u, the same element order as pack_vtq_tile)
            const int64_t nkt = (a.rowsVT + 63) / 64, ntv = a.nkbN * nkt;
            float* vt = smem_tiles + (size_t)a.r_slots * kPtW * (kPtW + 1);
            const int c = t & 63, g = t >> 6;
            for (int h0 = 0; h0 < a.hold_v; h0 += 2) {
                float x[2][16];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int64_t b = blockIdx.x + (int64_t)(h0 + hh) * gridDim.x;
                    const bool live = h0 + hh < a.hold_v && b < ntv;
                    const int64_t j0 = (b / nkt) * 64 + g, k = (b % nkt) * 64 + c;
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        x[hh][u] = live && j0 + 4 * u < a.N && k < a.r ? __ldg(a.V + (j0 + 4 * u) * a.r + k) : 0.f;
                }
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    if (h0 + hh >= a.hold_v) break;
                    float(*tl)[kPtW + 1] = reinterpret_cast<float(*)[kPtW + 1]>(vt + (size_t)(h0 + hh) * kPtW * (kPtW + 1));
                    float mx = 0.f;
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        tl[g + 4 * u][c] = x[hh][u];
                        mx = fmaxf(mx, fabsf(x[hh][u]));
                    }
                    cpart[hh][g][c] = mx;
                }
                __syncthreads();
                if (a.colmax && t < 128) {
                    const int hh = t >> 6;
                    const int64_t b = blockIdx.x + (int64_t)(h0 + hh) * gridDim.x;
                    const int64_t k = (b % nkt) * 64 + c;
                    const float mc = fmaxf(fmaxf(cpart[hh][0][c], cpart[hh][1][c]), fmaxf(cpart[hh][2][c], cpart[hh][3][c]));
                    if (h0 + hh < a.hold_v && b < ntv && k < a.r && mc > 0.f) atomicMax(a.vcol + k, __float_as_uint(mc));
                }
                __syncthreads();  // cpart reused
            }
        } else if (a.colmax) {
            // tile (64 rows of V) x (64 columns): thread = (column t & 63, 16-row group t >> 6)
            const int64_t nkc = (a.r + 63) / 64;
            const int c = t & 63, g = t >> 6;
            for (int64_t b = blockIdx.x; b < a.nkbN * nkc; b += gridDim.x) {
                const int64_t j0 = (b / nkc) * 64 + g * 16, k = (b % nkc) * 64 + c;
                float mx = 0.f;
                if (k < a.r) {
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (j0 + e < a.N) mx = fmaxf(mx, fabsf(a.V[(j0 + e) * a.r + k]));
                }
                tile0[g][c] = mx;
                __syncthreads();
                if (t < 64) {
                    const float mc = fmaxf(fmaxf(tile0[0][t], tile0[1][t]), fmaxf(tile0[2][t], tile0[3][t]));
                    const int64_t kk = (b % nkc) * 64 + t;
                    if (kk < a.r && mc > 0.f) atomicMax(a.vcol + kk, __float_as_uint(mc));
                }
                __syncthreads();
            }
        }
    }
    MID_MARK(1);
    grid.sync();
    MID_MARK(2);
    // ---- B: every block sums the partials in the same order (deterministic, no
    // extra barrier); the last block publishes them for the kernels after k_mid
    __shared__ double tot_s[2];
    {
        // all threads load the partials at once (a lane-strided loop in one warp was a
        // chain of dependent L2 round trips, ~5 us at 592 blocks)
        double l = 0.0, pn = 0.0;
#pragma unroll 4
        for (int b = t; b < (int)gridDim.x; b += kMidThreads) {
            l += a.part[2 * b];
            pn += a.part[2 * b + 1];
        }
        l = warp_sum(l);
        pn = warp_sum(pn);
        if (lane == 0) { red[0][w] = l; red[1][w] = pn; }  // red's phase-A readers passed the grid barrier
        __syncthreads();
        if (w == 0) {
            l = lane < kMidThreads / 32 ? red[0][lane] : 0.0;
            pn = lane < kMidThreads / 32 ? red[1][lane] : 0.0;
            l = warp_sum(l);
            pn = warp_sum(pn);
            if (lane == 0) {
                tot_s[0] = l;
                tot_s[1] = pn;
                if (blockIdx.x == gridDim.x - 1) {  // read by the kernels after k_mid
                    a.sc->loss = l;
                    a.sc->pnorm2 = pn;
                }
            }
        }
    }
    __syncthreads();
    MID_MARK(6);
    const bool stopped = tol > 0.0 && tot_s[0] <= tol * tot_s[1];
    const int64_t npairs = a.nkbN * (a.nkbN + 1) / 2;
    {
        const int64_t nkt = (a.rowsVT + 63) / 64, ntv = a.nkbN * nkt;
        if (a.hold_v) {
            // the V tiles held since phase A; thread = (VTQ row k0 + (t >> 2), 16-row chunk t & 3).
            // vcol took atomics in phase A: plain loads, all issued before the slicing
            const float* vt = smem_tiles + (size_t)a.r_slots * kPtW * (kPtW + 1);
            const int kk = t >> 2, c = t & 3;
            float sc[kMidMaxHeldV];
#pragma unroll
            for (int h = 0; h < kMidMaxHeldV; ++h) {
                const int64_t b = blockIdx.x + (int64_t)h * gridDim.x, k = (b % nkt) * 64 + kk;
                sc[h] = h < a.hold_v && b < ntv && k < a.r ? slice_scale(a.vcol[k]) : 0.f;
            }
#pragma unroll
            for (int h = 0; h < kMidMaxHeldV; ++h) {
                const int64_t b = blockIdx.x + (int64_t)h * gridDim.x;
                if (h >= a.hold_v || b >= ntv) break;
                const int64_t k = (b % nkt) * 64 + kk;
                if (k >= a.rowsVT) continue;
                const float(*tl)[kPtW + 1] = reinterpret_cast<const float(*)[kPtW + 1]>(vt + (size_t)h * kPtW * (kPtW + 1));
                float xs[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) xs[u] = tl[c * 16 + u][kk];
                uint4 q[3];
                slice16(xs, sc[h], q);
                store_q16(a.VTQ, b / nkt, k, c, a.nkbN, a.rowsVT, q);
            }
        } else {
            for (int64_t b = blockIdx.x; b < ntv; b += gridDim.x)
                pack_vtq_tile<256>(a.V, a.N, a.r, a.rowsVT, a.nkbN, a.vcol, a.VTQ, b / nkt, (b % nkt) * 64, tile0, t);
        }
    }
    MID_MARK(7);
    if (!stopped) {
        int slot = 0;
        for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++slot) {
            int64_t I, J;
            block_pair(pr, I, J);
            float* tile = a.hold ? smem_tiles + slot * kPtW * (kPtW + 1) : &tile0[0][0];
            gather_r_tile(a.pt, a.res, I, J, tile, t);
            __syncthreads();
            const int line = t >> 2, part = t & 3;
            float x[16];
            rt_row16<kGatherRows>(tile, line, part, x);
            float mr = 0.f, mc = 0.f;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                mr = fmaxf(mr, fabsf(x[e]));
                mc = fmaxf(mc, fabsf(rt_at<kGatherRows>(tile, part * 16 + e, line)));
            }
            mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 1));
            mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, 2));
            mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 1));
            mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 2));
            if (part == 0) {
                if (mr > 0.f) atomicMax(a.rrow + I * kPtW + line, __float_as_uint(mr));
                if (I != J && mc > 0.f) atomicMax(a.rrow + J * kPtW + line, __float_as_uint(mc));
            }
            if (!a.hold) __syncthreads();  // tile0 is reused by the next block pair
        }
    }
    MID_MARK(8);
    for (int64_t e = gtid; e < a.M / 4; e += gstride) reinterpret_cast<float4*>(a.coef)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = (a.M / 4) * 4 + gtid; e < a.M; e += gstride) a.coef[e] = 0.f;
    // t += 1 and the loss record, once per step (nothing in k_mid reads them)
    auto step_record = [&]() {
        if (blockIdx.x == gridDim.x - 1 && t == 0) {
            advance_step(a.opt);
            double* L = a.losses_from_opt ? a.opt->losses : a.losses;
            if (L) L[a.losses_from_opt ? a.opt->loss_idx++ : 0] = tot_s[0];
        }
    };
    if (stopped) {  // grid-uniform: every block leaves before the barrier
        step_record();
        return;
    }
    MID_MARK(3);
    grid.sync();
    MID_MARK(4);
    // ---- C: slice the held blocks (or, when they do not fit, gather them again)
    int slot = 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++slot) {
        int64_t I, J;
        block_pair(pr, I, J);
        float* tile = a.hold ? smem_tiles + slot * kPtW * (kPtW + 1) : &tile0[0][0];
        if (!a.hold) {
            gather_r_tile(a.pt, a.res, I, J, tile, t);
            __syncthreads();
        }
        const int rr = t >> 2, c = t & 3;
        float x[16];
        uint4 q[3];
        rt_row16<kGatherRows>(tile, rr, c, x);
        slice16(x, slice_scale(a.rrow[I * kPtW + rr]), q);
        store_q16(a.RQ, J, I * kPtW + rr, c, a.nkbN, a.Np, q);
        if (I != J) {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = rt_at<kGatherRows>(tile, c * 16 + e, rr);
            slice16(x, slice_scale(a.rrow[J * kPtW + rr]), q);
            store_q16(a.RQ, I, J * kPtW + rr, c, a.nkbN, a.Np, q);
        }
        if (!a.hold) __syncthreads();
    }
    step_record();
    MID_MARK(5);
#ifdef SOS_EXPERIMENTS
    if (a.trace && blockIdx.x == 0 && t == 0)
        printf("k_mid block0 (us): A %.2f | sync %.2f | B %.2f | sync %.2f | C %.2f\n", (tmark[1] - tmark[0]) * 1e-3,
               (tmark[2] - tmark[1]) * 1e-3, (tmark[3] - tmark[2]) * 1e-3, (tmark[4] - tmark[3]) * 1e-3,
               (tmark[5] - tmark[4]) * 1e-3);
    if (a.trace && blockIdx.x == 0 && t == 0)
        printf("k_mid block0 detail (us): A residual %.2f | B partials %.2f | B vtq %.2f | B r-gather %.2f | B coef0 %.2f\n",
               (tmark[9] - tmark[0]) * 1e-3, (tmark[6] - tmark[2]) * 1e-3, (tmark[7] - tmark[6]) * 1e-3,
               (tmark[8] - tmark[7]) * 1e-3, (tmark[3] - tmark[8]) * 1e-3);
    if (a.trace && a.dbg) {  // slowest block per phase: (ns << 16) | block
        const unsigned long long id = blockIdx.x;
        if (t == 0) {
            atomicMax(a.dbg + 0, ((tmark[1] - tmark[0]) << 16) | id);
            atomicMax(a.dbg + 1, ((tmark[3] - tmark[2]) << 16) | id);
            atomicMax(a.dbg + 2, ((tmark[7] - tmark[6]) << 16) | id);
            atomicMax(a.dbg + 3, ((tmark[8] - tmark[7]) << 16) | id);
            atomicMax(a.dbg + 4, ((tmark[5] - tmark[4]) << 16) | id);
            atomicMax(a.dbg + 5, ((tmark[9] - tmark[0]) << 16) | id);
        }
        grid.sync();
        if (blockIdx.x == 0 && t == 0) {
            const char* nm[6] = {"A", "B", "B vtq", "B r-gather", "C", "A residual"};
            printf("k_mid slowest blocks (us@block):");
            for (int k = 0; k < 6; ++k) printf(" %s %.2f@%llu |", nm[k], (a.dbg[k] >> 16) * 1e-3, a.dbg[k] & 0xffff);
            printf(" grid %d hold_v %d r_slots %d\n", (int)gridDim.x, a.hold_v, a.r_slots);
        }
    }
#endif
}

// cooperative grid of k_mid: no more blocks than work items of its largest phase
// (a grid barrier costs more with more blocks), at most 4 per SM, and every
// block holds ceil(npairs / grid) R blocks in shared memory -- or, when that
// exceeds kMidMaxHeld (long K), one block at a time with phase C gathering
// again (tiles_per_block = 0).  Returns the grid (blocks).
int mid_grid_for(int64_t nkbN, int64_t rowsVT, int64_t M, int num_sms, int* tiles_per_block, int* hold_v) {
    const int64_t npairs = nkbN * (nkbN + 1) / 2;
    const int64_t ntv = nkbN * ((rowsVT + 63) / 64);
    const int64_t work = std::max<int64_t>({npairs, ntv, (M + 1023) / 1024, 1});
    auto blocks_per_sm = [&](size_t smem) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_mid, kMidThreads, smem) != cudaSuccess || nb < 1) {
            cudaGetLastError();
            nb = 1;
        }
        return std::min(nb, 4);
    };
    auto grid_for_smem = [&](size_t smem) { return (int)std::min<int64_t>(work, (int64_t)num_sms * blocks_per_sm(smem)); };
    int tpb = 1, grid = grid_for_smem(kMidTileBytes);
    *hold_v = 0;
    for (int it = 0; it < 8; ++it) {
        const int need = (int)((npairs + grid - 1) / grid);
        if (need <= tpb) break;
        if (need > kMidMaxHeld) {  // R does not fit: hold nothing
            *tiles_per_block = 0;
            return grid_for_smem(kMidTileBytes);
        }
        tpb = need;
        grid = grid_for_smem((size_t)tpb * kMidTileBytes);
    }
    *tiles_per_block = tpb;
    // the V tiles of phase A held for phase B, when they fit beside the R blocks
    // without shrinking the grid
    const int hv = (int)((ntv + grid - 1) / grid);
    if (hv <= kMidMaxHeldV && (int64_t)num_sms * blocks_per_sm((size_t)(tpb + hv) * kMidTileBytes) >= grid) *hold_v = hv;
    blocks_per_sm((size_t)(tpb + *hold_v) * kMidTileBytes);  // leaves the attribute at the launch's size
    return grid;
}

void launch_mid(Plan& P, const float* p, const float* V, unsigned* vcol, bool colmax, unsigned* zero_cols,
                double* losses, bool losses_from_opt, cudaStream_t st) {
    LaunchScope ls(P, KK_MID, st);
    MidArgs a;
    a.coef = P.d_coef;
    a.p = p;
    a.res = P.d_res;
    a.M = P.idx->M;
    a.sc = P.d_scal;
    a.opt = P.d_opt;
    a.losses = losses;
    a.losses_from_opt = losses_from_opt ? 1 : 0;
    a.pt = P.idx->d_pt;
    a.Np = P.idx->Np;
    a.nkbN = P.nkbN;
    a.rrow = P.d_rrow;
    a.RQ = P.d_rq;
    a.V = V;
    a.N = P.idx->N;
    a.r = P.r;
    a.rowsVT = P.rowsVT;
    a.vcol = vcol;
    a.colmax = colmax ? 1 : 0;
    a.VTQ = P.d_vtq;
    a.zero_cols = zero_cols;
    a.part = P.d_part;
    a.trace = 0;
    a.dbg = nullptr;
#ifdef SOS_EXPERIMENTS
    {
        const char* e = getenv("SOS_MID_TRACE");
        a.trace = e && atoi(e) ? 1 : 0;
        static unsigned long long* dbg = nullptr;
        if (a.trace && !dbg) cudaMalloc(&dbg, 8 * sizeof(unsigned long long));
        if (a.trace) cudaMemsetAsync(dbg, 0, 8 * sizeof(unsigned long long), st);
        a.dbg = dbg;
    }
#endif
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.mid_grid);
    cfg.blockDim = dim3(kMidThreads);
    a.hold = P.mid_tiles > 0 ? 1 : 0;
    a.r_slots = std::max(P.mid_tiles, 1);
    a.hold_v = P.mid_hold_v;
    cfg.dynamicSmemBytes = (size_t)(a.r_slots + a.hold_v) * kMidTileBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ls.a ? 1 : 2;
    if (cudaLaunchKernelEx(&cfg, k_mid, a) != cudaSuccess && cfg.numAttrs == 2) {
        cudaGetLastError();
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_mid, a);
    }
}

void launch_step_begin(Plan& P, double* losses, cudaStream_t st, bool losses_from_opt, unsigned* zero0, int64_t n0,
                       unsigned* zero1, int64_t n1, float* zero_coef, unsigned* zero_r) {
    LaunchScope ls(P, KK_UPDATE, st);
    const int64_t nc = zero_coef ? P.idx->M : 0;
    const int64_t n2 = zero_r ? P.idx->Np : 0;
    if (!zero0) n0 = 0;
    if (!zero1) n1 = 0;
    const int64_t nz = n0 + n1 + n2;
    const int blocks = nz || nc ? grid_for(P, k_step_begin, std::max<int64_t>(nz, nc / 4), 256, 4) : 1;
    k_step_begin<<<blocks, 256, 0, st>>>(P.d_opt, P.d_scal, losses_from_opt ? nullptr : losses, losses_from_opt ? 1 : 0,
                                         zero0, n0, zero1, n1, zero_r, n2, zero_coef, nc);
}

// maxima (one read of V) + VQ (one elementwise pass)
void launch_pack_v(Plan& P, const float* V, cudaStream_t st, unsigned* vrow, unsigned* vcol) {
    if (!vrow) vrow = P.d_vrow;
    launch_vmax(P, V, st, vrow, vcol);
    LaunchScope ls(P, KK_PACK_V, st);
    const int64_t work = P.rowsV * P.nkbV * 4;
    k_pack_vq<<<grid_for(P, k_pack_vq, work, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.rowsV, P.nkbV, vrow, P.d_vq);
}

// row maxima + RQ: the row maxima come from the lattice DP (sos_index.cu, a
// few tens of millions of lookups instead of N^2 gathers) or the direct pass,
// then one streaming pass gathers and slices R.
// R row maxima: the lattice DP costs ~d launches plus sum_D C(n+D-1, D) * n
// lookups; the direct pass over the stored PT triangle (k_rmax) a memset, one
// launch and N^2 / 2 lookups.
// Small problems and many variables favour the direct pass (config 2: 60 -> 14
// us; N = 5050 quartic: 100 -> 32 us); config 4 the DP (0.33 vs 0.46 ms); config
// 3 is even (0.178 / 0.175 ms).  Rates fitted to those measurements.
bool rmax_direct_default(const Index& ix) {
    double lookups = 0;
    for (int D = ix.d; D <= 2 * ix.d - 1; ++D) lookups += (double)rmax_level_count(ix.n, D) * ix.n;
    const double dp_us = 12.0 * ix.d + lookups / 2e5;
    const double direct_us = 6.0 + (double)ix.N * ix.N / 9e5;  // per stored block pair (k_rmax)
    return direct_us < dp_us;
}

void launch_pack_r(Plan& P, const float* res, cudaStream_t st, int use_stop, bool rrow_zeroed) {
    if (P.rmax_direct) {
        launch_rmax(P, res, st, use_stop, rrow_zeroed);
    } else {
        LaunchScope ls(P, KK_ABSMAX_R, st);
        launch_rmax_dp(*P.idx, res, P.d_rlev, P.d_rrow, st, P.d_scal, P.d_opt, use_stop);
        P.launches += P.idx->d - 1;  // one kernel per lattice level (the scope counts one)
    }
    launch_pack_rq(P, res, st, use_stop);
}

void launch_pack_rq(Plan& P, const float* res, cudaStream_t st, int use_stop) {
    const int64_t Np = P.idx->Np;
    LaunchScope ls(P, KK_PACK_R, st);
    const int64_t npairs = P.nkbN * (P.nkbN + 1) / 2;
    const unsigned blocks = grid_for(P, k_pack_rq_sym<false>, npairs * 256, 256);
    k_pack_rq_sym<false><<<blocks, 256, 0, st>>>(P.idx->d_pt, res, Np, P.nkbN, P.d_rrow, P.d_rq, P.d_scal, P.d_opt,
                                                 use_stop, nullptr);
}

void launch_pack_r_headroom(Plan& P, const float* res, const unsigned* rrow_prev, unsigned* rrow_cur,
                            unsigned* urow_r, cudaStream_t st) {
    const int64_t Np = P.idx->Np;
    {
        LaunchScope ls(P, KK_PACK_R, st);
        const int64_t npairs = P.nkbN * (P.nkbN + 1) / 2;
        const unsigned blocks = grid_for(P, k_pack_rq_sym<true>, npairs * 256, 256);
        k_pack_rq_sym<true><<<blocks, 256, 0, st>>>(P.idx->d_pt, res, Np, P.nkbN, rrow_prev, P.d_rq, P.d_scal,
                                                    P.d_opt, 1, rrow_cur);
    }
    LaunchScope ls(P, KK_ABSMAX_R, st);
    k_rfix<<<grid_for(P, k_rfix, P.idx->N * 32, 256), 256, 0, st>>>(P.idx->d_pt, res, P.idx->N, Np, P.nkbN, rrow_prev,
                                                              rrow_cur, urow_r, P.d_rq, P.d_scal, P.d_opt);
}


// ------------------------------------------------------- sos_descend fixup --
// Before the forward of step t+1 (long K, fused update): the update of step t
// wrote the slices of each updated row of V with the scale kHeadroom * (row
// max of V_t), and (vtq_from_update) the V^T slices of each column with
// kHeadroom * (column max of V_t).  They stay exact to ~22 bits while the new
// maximum lies in [u/4, u], u = kHeadroom * old max; the rare rows / columns
// outside (growth beyond the headroom, or a large shrink) are re-sliced here
// from V with their exact new maximum, and urow_next / ucol_next receive the
// scale each row / column was written with.  One warp per row, then one warp
// per column (cols != 0), in a single launch: the common case is one load and
// one store per warp.  If the stopping rule held at step t the update did not
// run and everything of step t carries over.
struct FixupArgs {
    const float* V;
    int64_t N, r, rowsV, nkbV, rowsVT, nkbN;
    const unsigned *vrow_cur, *urow_cur, *vcol_cur;
    unsigned *vrow_next, *urow_next, *vcol_next, *ucol_next;
    uint8_t* VQ;
    uint8_t* VTQ;  // nullptr: no column fixup (the forward packs V^T)
    const Scalars* sc;
    const DevOpt* opt;
};
__global__ void __launch_bounds__(256) k_descend_fixup(const FixupArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (descent_stopped(a.sc, a.opt, 1)) {
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.rowsV; e += stride) {
            a.vrow_next[e] = a.vrow_cur[e];
            a.urow_next[e] = a.urow_cur[e];
        }
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.rowsVT; e += stride)
            a.vcol_next[e] = a.vcol_cur[e];
        return;
    }
    const int64_t nrow = a.rowsV, ncol = a.VTQ ? a.r : 0;
    for (int64_t w = warp; w < nrow + ncol; w += nwarps) {
        if (w < nrow) {
            const int64_t i = w;
            const float u = kHeadroom * __uint_as_float(a.vrow_cur[i]);
            const unsigned mb = a.vrow_next[i];
            const float mx = __uint_as_float(mb);
            const bool keep = mx <= u && mx >= 0.25f * u;
            if (lane == 0) a.urow_next[i] = keep ? __float_as_uint(u) : mb;
            if (keep) continue;
            const float c = slice_scale(mb);
            for (int64_t cc = lane; cc < a.nkbV * 4; cc += 32) {
                const int64_t k0 = cc * 16;
                float x[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) x[e] = (i < a.N && k0 + e < a.r) ? a.V[i * a.r + k0 + e] : 0.f;
                uint4 q[3];
                slice16(x, c, q);
                store_q16(a.VQ, cc >> 2, i, (int)(cc & 3), a.nkbV, a.rowsV, q);
            }
        } else {
            const int64_t k = w - nrow;
            const float u = kHeadroom * __uint_as_float(a.vcol_cur[k]);
            const unsigned mb = a.vcol_next[k];
            const float mx = __uint_as_float(mb);
            const bool keep = mx <= u && mx >= 0.25f * u;
            if (lane == 0) a.ucol_next[k] = keep ? __float_as_uint(u) : mb;
            if (keep) continue;
            const float c = slice_scale(mb);
            for (int64_t cc = lane; cc < a.nkbN * 4; cc += 32) {
                const int64_t j0 = cc * 16;
                float x[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) x[e] = j0 + e < a.N ? a.V[(j0 + e) * a.r + k] : 0.f;
                uint4 q[3];
                slice16(x, c, q);
                store_q16(a.VTQ, cc >> 2, k, (int)(cc & 3), a.nkbN, a.rowsVT, q);
            }
        }
    }
}

void launch_descend_fixup(Plan& P, const float* V, const unsigned* vrow_cur, unsigned* vrow_next,
                          const unsigned* urow_cur, unsigned* urow_next, const unsigned* vcol_cur, unsigned* vcol_next,
                          unsigned* ucol_next, uint8_t* vtq_next, cudaStream_t st) {
    LaunchScope ls(P, KK_PACK_V, st);
    FixupArgs a;
    a.V = V;
    a.N = P.idx->N;
    a.r = P.r;
    a.rowsV = P.rowsV;
    a.nkbV = P.nkbV;
    a.rowsVT = P.rowsVT;
    a.nkbN = P.nkbN;
    a.vrow_cur = vrow_cur;
    a.urow_cur = urow_cur;
    a.vcol_cur = vcol_cur;
    a.vrow_next = vrow_next;
    a.urow_next = urow_next;
    a.vcol_next = vcol_next;
    a.ucol_next = ucol_next;
    a.VQ = P.d_vq;
    a.VTQ = vtq_next;
    a.sc = P.d_scal;
    a.opt = P.d_opt;
    const int64_t warps = P.rowsV + (vtq_next ? P.r : 0);
    k_descend_fixup<<<grid_for(P, k_descend_fixup, warps * 32, 256), 256, 0, st>>>(a);
}

}  // namespace sos

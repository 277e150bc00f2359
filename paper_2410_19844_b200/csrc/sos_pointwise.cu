// sos_pointwise.cu -- HBM-bound kernels of the step: per-row maxima and int8
// slice packing of V, V^T and of the residual matrix R (R_ij = res[rank(alpha_i +
// alpha_j)], gathered through the pair-rank table), and the fused residual +
// loss reduction.  The optimiser update of PAPER.md:221 runs inside the backward
// GEMM (sos_gemmq.cu).  All kernels are coalesced and sized as a multiple of
// the SM count (grid-stride).
#include <algorithm>
#include <cstdlib>

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
        pack_vtq_tile(V, N, r, rowsVT, nkbN, vcol, VTQ, b / nkt, (b % nkt) * 64, tile, threadIdx.x, 256);
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
    __shared__ float tile[kPtW][kPtW + 1];
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
            const int e = (u * 256 + t) * 4;
            const uint4 k = __ldg(reinterpret_cast<const uint4*>(p0 + e));
            float* d = &tile[e >> 6][e & 63];
            d[0] = k.x != kInvalidRank ? fabsf(__ldg(res + k.x)) : 0.f;
            d[1] = k.y != kInvalidRank ? fabsf(__ldg(res + k.y)) : 0.f;
            d[2] = k.z != kInvalidRank ? fabsf(__ldg(res + k.z)) : 0.f;
            d[3] = k.w != kInvalidRank ? fabsf(__ldg(res + k.w)) : 0.f;
        }
        __syncthreads();
        // thread t: row (t & 63) of the block if t < 64 ... four threads per line
        const int line = t >> 2, part = t & 3;
        float mr = 0.f, mc = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            mr = fmaxf(mr, tile[line][part * 16 + e]);   // row `line` of I
            mc = fmaxf(mc, tile[part * 16 + e][line]);   // column `line` = row of J
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
__global__ void __launch_bounds__(256, 6) k_pack_rq_sym(const uint32_t* __restrict__ pt, const float* __restrict__ res,
                                                     int64_t Np, int64_t nkb, const unsigned* __restrict__ rrow,
                                                     uint8_t* __restrict__ RQ, const Scalars* sc, const DevOpt* opt,
                                                     int use_stop) {
    if (descent_stopped(sc, opt, use_stop)) return;
    __shared__ float tile[kPtW][kPtW + 1];  // [row in I][j in J], padded
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
            const int e = (u * 256 + t) * 4;
            const uint4 k = __ldg(reinterpret_cast<const uint4*>(p0 + e));
            float* d = &tile[e >> 6][e & 63];
            d[0] = k.x != kInvalidRank ? __ldg(res + k.x) : 0.f;
            d[1] = k.y != kInvalidRank ? __ldg(res + k.y) : 0.f;
            d[2] = k.z != kInvalidRank ? __ldg(res + k.z) : 0.f;
            d[3] = k.w != kInvalidRank ? __ldg(res + k.w) : 0.f;
        }
        __syncthreads();
        const int r = t >> 2, c = t & 3;
        float x[16];
        uint4 q[3];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = tile[r][c * 16 + e];
        slice16(x, slice_scale(__ldg(rrow + I * kPtW + r)), q);
        store_q16(RQ, J, I * kPtW + r, c, nkb, Np, q);
        if (I != J) {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = tile[c * 16 + e][r];
            slice16(x, slice_scale(__ldg(rrow + J * kPtW + r)), q);
            store_q16(RQ, I, J * kPtW + r, c, nkb, Np, q);
        }
        __syncthreads();
    }
}


// -------------------------------------------------------------- launches ---
static int grid_for(const Plan& P, int64_t work, int threads, int per_sm = 8) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = (int64_t)P.num_sms * per_sm;
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
    k_vmax<<<grid_for(P, tiles * 256, 256), 256, 0, st>>>(V, N, P.r, vrow, vcol);
}

void launch_pack_vtq(Plan& P, const float* V, cudaStream_t st, const unsigned* vcol) {
    LaunchScope ls(P, KK_PACK_V, st);
    const int64_t blocks = P.nkbN * ((P.rowsVT + 63) / 64);
    k_pack_vtq<<<grid_for(P, blocks * 256, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.rowsVT, P.nkbN,
                                                               vcol ? vcol : P.d_vcol, P.d_vtq);
}

void launch_residual(Plan& P, const float* coef, const float* p, float* res, cudaStream_t st) {
    LaunchScope ls(P, KK_RESIDUAL, st);
    k_residual<<<grid_for(P, P.idx->M, 256, 4), 256, 0, st>>>(coef, p, res, P.idx->M, P.d_scal);
}

void launch_rmax(Plan& P, const float* res, cudaStream_t st, int use_stop) {
    LaunchScope ls(P, KK_ABSMAX_R, st);
    cudaMemsetAsync(P.d_rrow, 0, (size_t)P.idx->Np * sizeof(unsigned), st);
    const int64_t nkb = P.idx->Np / kPtW, npairs = nkb * (nkb + 1) / 2;
    const unsigned blocks = (unsigned)std::min<int64_t>(npairs, (int64_t)P.num_sms * 8);
    k_rmax<<<blocks, 256, 0, st>>>(P.idx->d_pt, res, nkb, P.d_rrow, P.d_scal, P.d_opt, use_stop);
}

// one thread: t += 1 (Adam bias correction of this step), and in sos_descend
// the loss of this step into the caller's array
// step bookkeeping (Adam t, loss record) and, inside sos_descend, zeroing of
// the next step's maxima accumulators (zero0 / zero1: n0 / n1 words) and of
// the coefficient accumulator of the next forward (zc: nc floats, 16-B aligned)
__global__ void k_step_begin(DevOpt* opt, const Scalars* sc, double* losses, int from_opt, unsigned* zero0,
                             int64_t n0, unsigned* zero1, int64_t n1, float* zc, int64_t nc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        opt->t += 1;
        if (from_opt) losses = opt->losses;
        if (losses) losses[opt->loss_idx++] = sc->loss;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t e = tid; e < n0 + n1; e += stride) {
        if (e < n0) zero0[e] = 0u;
        else zero1[e - n0] = 0u;
    }
    for (int64_t e = tid; e < nc / 4; e += stride) reinterpret_cast<float4*>(zc)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = (nc / 4) * 4 + tid; e < nc; e += stride) zc[e] = 0.f;
}

// The optimiser step over the whole N x r gradient (short-K problems, see
// Plan::update_split).  Block tile = 16 rows x 256 columns: warp w owns rows
// 2w, 2w+1, lane l the columns l + 32e (e < 8), so every access is a coalesced
// row segment and all 64 loads of a thread are in flight together; the new
// values are staged in shared memory for the next step's VQ chunks (task =
// row x 16-column chunk, scale kHeadroom * old row max); row maxima by warp
// shuffles, column maxima per thread over its rows, then across the 8 warps.
constexpr int kUpdCols = 256, kUpdLd = kUpdCols + 4;
__global__ void __launch_bounds__(256) k_update(const float* __restrict__ grad, float* __restrict__ V,
                                                float* __restrict__ m, float* __restrict__ v, int64_t N, int64_t r,
                                                int adam, const DevOpt* opt, const Scalars* sc,
                                                uint8_t* __restrict__ vq_next, int64_t rowsV, int64_t nkbV,
                                                const unsigned* __restrict__ vrow_cur, unsigned* __restrict__ vrow_next,
                                                unsigned* __restrict__ vcol_next) {
    if (descent_stopped(sc, opt, 1)) return;
    constexpr int kE = kUpdCols / 32;
    __shared__ float cst[6];
    __shared__ __align__(16) float stage[16 * kUpdLd];
    __shared__ float cm_s[8][kUpdCols];
    if (threadIdx.x == 0) {
        const DevOpt o = *opt;
        cst[0] = o.lr;
        cst[1] = o.b1;
        cst[2] = o.b2;
        cst[3] = o.eps;
        cst[4] = (float)((double)o.lr / (1.0 - pow((double)o.b1, (double)o.t)));
        cst[5] = (float)(1.0 / sqrt(1.0 - pow((double)o.b2, (double)o.t)));
    }
    __syncthreads();
    const float lr = cst[0], b1 = cst[1], b2 = cst[2], eps = cst[3], lr_c1 = cst[4], isc2 = cst[5];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, t = threadIdx.x;
    const bool q = vq_next != nullptr;
    const int64_t col_tiles = (r + kUpdCols - 1) / kUpdCols, row_tiles = (N + 15) / 16;
    for (int64_t blk = blockIdx.x; blk < row_tiles * col_tiles; blk += gridDim.x) {
        const int64_t row0 = (blk / col_tiles) * 16, col0 = (blk % col_tiles) * kUpdCols;
        float gv[2][kE], x[2][kE], mm[2][kE], vv[2][kE];
        bool ok[2][kE];
        int64_t ro[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int64_t i = row0 + 2 * w + k;
            ro[k] = i * r + col0 + lane;
#pragma unroll
            for (int e = 0; e < kE; ++e) {
                ok[k][e] = i < N && col0 + lane + 32 * e < r;
                gv[k][e] = ok[k][e] ? grad[ro[k] + 32 * e] : 0.f;
                x[k][e] = ok[k][e] ? V[ro[k] + 32 * e] : 0.f;
                if (adam) {
                    mm[k][e] = ok[k][e] ? m[ro[k] + 32 * e] : 0.f;
                    vv[k][e] = ok[k][e] ? v[ro[k] + 32 * e] : 0.f;
                }
            }
        }
        float cm[kE];
#pragma unroll
        for (int e = 0; e < kE; ++e) cm[e] = 0.f;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float mx = 0.f;
#pragma unroll
            for (int e = 0; e < kE; ++e) {
                float xn = 0.f;
                if (ok[k][e]) {
                    if (adam) {
                        mm[k][e] = b1 * mm[k][e] + (1.f - b1) * gv[k][e];
                        vv[k][e] = b2 * vv[k][e] + (1.f - b2) * gv[k][e] * gv[k][e];
                        xn = x[k][e] - lr_c1 * mm[k][e] / (sqrtf(vv[k][e]) * isc2 + eps);
                        m[ro[k] + 32 * e] = mm[k][e];
                        v[ro[k] + 32 * e] = vv[k][e];
                    } else {
                        xn = x[k][e] - lr * gv[k][e];
                    }
                    V[ro[k] + 32 * e] = xn;
                }
                if (q) {
                    stage[(2 * w + k) * kUpdLd + lane + 32 * e] = xn;
                    mx = fmaxf(mx, fabsf(xn));
                    cm[e] = fmaxf(cm[e], fabsf(xn));
                }
            }
            if (q) {
                mx = warp_max(mx);
                const int64_t i = row0 + 2 * w + k;
                if (lane == 0 && i < N && mx > 0.f) atomicMax(vrow_next + i, __float_as_uint(mx));
            }
        }
        if (q) {
#pragma unroll
            for (int e = 0; e < kE; ++e) cm_s[w][lane + 32 * e] = cm[e];
            __syncthreads();
            {   // task t = (row t / 16, 16-column chunk t % 16)
                const int rr = t >> 4, cq = t & 15;
                const int64_t i = row0 + rr, k0 = col0 + 16 * cq;
                if (i < N && k0 < r) {
                    float xs[16];
                    const float4* s4 = reinterpret_cast<const float4*>(stage + rr * kUpdLd + 16 * cq);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 f = s4[q4];
                        xs[4 * q4] = f.x; xs[4 * q4 + 1] = f.y; xs[4 * q4 + 2] = f.z; xs[4 * q4 + 3] = f.w;
                    }
                    const float um = kHeadroom * __uint_as_float(__ldg(vrow_cur + i));
                    uint4 qq[3];
                    slice16(xs, slice_scale(__float_as_uint(um)), qq);
                    store_q16(vq_next, k0 >> 6, i, (int)((k0 >> 4) & 3), nkbV, rowsV, qq);
                }
            }
            {   // column t: maximum over the 16 rows (8 warps x 2)
                float c = 0.f;
#pragma unroll
                for (int ww = 0; ww < 8; ++ww) c = fmaxf(c, cm_s[ww][t]);
                if (col0 + t < r && c > 0.f) atomicMax(vcol_next + col0 + t, __float_as_uint(c));
            }
            __syncthreads();
        }
    }
}

void launch_update_split(Plan& P, float* V, cudaStream_t st, const DescendBufs* db) {
    LaunchScope ls(P, KK_UPDATE, st);
    const int64_t N = P.idx->N, blocks = ((N + 15) / 16) * ((P.r + kUpdCols - 1) / kUpdCols);
    k_update<<<grid_for(P, blocks * 256, 256), 256, 0, st>>>(
        P.d_grad, V, P.d_m, P.d_v, N, P.r, P.opt_kind == 1, P.d_opt, P.d_scal, db ? P.d_vq : nullptr, P.rowsV,
        P.nkbV, db ? db->vrow_cur : nullptr, db ? db->vrow_next : nullptr, db ? db->vcol_next : nullptr);
}

void launch_step_begin(Plan& P, double* losses, cudaStream_t st, bool losses_from_opt, unsigned* zero0, int64_t n0,
                       unsigned* zero1, int64_t n1, float* zero_coef) {
    LaunchScope ls(P, KK_UPDATE, st);
    const int64_t nc = zero_coef ? P.idx->M : 0;
    const int blocks = zero0 || zero1 || zero_coef ? grid_for(P, std::max<int64_t>(n0 + n1, nc / 4), 256, 4) : 1;
    k_step_begin<<<blocks, 256, 0, st>>>(P.d_opt, P.d_scal, losses_from_opt ? nullptr : losses, losses_from_opt ? 1 : 0,
                                         zero0, zero0 ? n0 : 0, zero1, zero1 ? n1 : 0, zero_coef, nc);
}

// maxima (one read of V) + VQ (one elementwise pass)
void launch_pack_v(Plan& P, const float* V, cudaStream_t st, unsigned* vrow, unsigned* vcol) {
    if (!vrow) vrow = P.d_vrow;
    launch_vmax(P, V, st, vrow, vcol);
    LaunchScope ls(P, KK_PACK_V, st);
    const int64_t work = P.rowsV * P.nkbV * 4;
    k_pack_vq<<<grid_for(P, work, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.rowsV, P.nkbV, vrow, P.d_vq);
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
static bool rmax_direct_is_cheaper(const Index& ix) {
    double lookups = 0;
    for (int D = ix.d; D <= 2 * ix.d - 1; ++D) lookups += (double)rmax_level_count(ix.n, D) * ix.n;
    const double dp_us = 12.0 * ix.d + lookups / 2e5;
    const double direct_us = 6.0 + (double)ix.N * ix.N / 9e5;  // per stored block pair (k_rmax)
    return direct_us < dp_us;
}

void launch_pack_r(Plan& P, const float* res, cudaStream_t st, int use_stop) {
    static const char* tp_env = getenv("SOS_RPACK_TWOPASS");
    if (tp_env ? atoi(tp_env) != 0 : rmax_direct_is_cheaper(*P.idx)) {
        launch_rmax(P, res, st, use_stop);
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
    const unsigned blocks = (unsigned)std::min<int64_t>(npairs, (int64_t)P.num_sms * 8);
    k_pack_rq_sym<<<blocks, 256, 0, st>>>(P.idx->d_pt, res, Np, P.nkbN, P.d_rrow, P.d_rq, P.d_scal, P.d_opt,
                                          use_stop);
}


// ------------------------------------------------------- sos_descend fixup --
// Before the forward of step t+1: the update of step t wrote the slices of each
// updated row with the scale kHeadroom * (row max of V_t).  They stay exact to
// ~22 bits while the new row max lies in [u/4, u], u = kHeadroom * old max; the
// rare rows outside (growth beyond the headroom, or a large shrink) are re-sliced
// here from V with their exact new maximum.  urow_next receives the scale the
// forward must use for every row.  If the stopping rule held at step t the
// update did not run, and everything of step t carries over.
__global__ void __launch_bounds__(256) k_descend_fixup(const float* __restrict__ V, int64_t N, int64_t r,
                                                       int64_t rowsV, int64_t nkbV, int64_t rowsVT,
                                                       const unsigned* __restrict__ vrow_cur,
                                                       unsigned* __restrict__ vrow_next,
                                                       const unsigned* __restrict__ urow_cur,
                                                       unsigned* __restrict__ urow_next,
                                                       const unsigned* __restrict__ vcol_cur,
                                                       unsigned* __restrict__ vcol_next, uint8_t* __restrict__ VQ,
                                                       const Scalars* sc, const DevOpt* opt) {
    if (descent_stopped(sc, opt, 1)) {
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rowsV; e += stride) {
            vrow_next[e] = vrow_cur[e];
            urow_next[e] = urow_cur[e];
        }
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rowsVT; e += stride)
            vcol_next[e] = vcol_cur[e];
        return;
    }
    for (int64_t i = blockIdx.x; i < rowsV; i += gridDim.x) {
        const float u = kHeadroom * __uint_as_float(vrow_cur[i]);
        const unsigned mb = vrow_next[i];
        const float mx = __uint_as_float(mb);
        if (mx <= u && mx >= 0.25f * u) {
            if (threadIdx.x == 0) urow_next[i] = __float_as_uint(u);
            continue;
        }
        if (threadIdx.x == 0) urow_next[i] = mb;
        const float c = slice_scale(mb);
        for (int64_t cc = threadIdx.x; cc < nkbV * 4; cc += blockDim.x) {
            const int64_t k0 = cc * 16;
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = (i < N && k0 + e < r) ? V[i * r + k0 + e] : 0.f;
            uint4 q[3];
            slice16(x, c, q);
            store_q16(VQ, cc >> 2, i, (int)(cc & 3), nkbV, rowsV, q);
        }
    }
}

// The same for the V^T slices the update wrote for step t+1 (scale kHeadroom x
// the old column maximum): a column whose new maximum left [u/4, u] is
// re-sliced from V with its exact maximum (strided reads: rare); ucol_next
// receives the scale the backward must unscale each VTQ row with.
__global__ void __launch_bounds__(256) k_descend_fixup_cols(const float* __restrict__ V, int64_t N, int64_t r,
                                                            int64_t nkbN, int64_t rowsVT,
                                                            const unsigned* __restrict__ vcol_cur,
                                                            const unsigned* __restrict__ vcol_next,
                                                            unsigned* __restrict__ ucol_next, uint8_t* __restrict__ VTQ,
                                                            const Scalars* sc, const DevOpt* opt) {
    if (descent_stopped(sc, opt, 1)) return;  // no update ran: the next step reads nothing new
    for (int64_t k = blockIdx.x; k < r; k += gridDim.x) {
        const float u = kHeadroom * __uint_as_float(vcol_cur[k]);
        const unsigned mb = vcol_next[k];
        const float mx = __uint_as_float(mb);
        if (mx <= u && mx >= 0.25f * u) {
            if (threadIdx.x == 0) ucol_next[k] = __float_as_uint(u);
            continue;
        }
        if (threadIdx.x == 0) ucol_next[k] = mb;
        const float c = slice_scale(mb);
        for (int64_t cc = threadIdx.x; cc < nkbN * 4; cc += blockDim.x) {
            const int64_t j0 = cc * 16;
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = j0 + e < N ? V[(j0 + e) * r + k] : 0.f;
            uint4 q[3];
            slice16(x, c, q);
            store_q16(VTQ, cc >> 2, k, (int)(cc & 3), nkbN, rowsVT, q);
        }
    }
}

void launch_descend_fixup_cols(Plan& P, const float* V, const unsigned* vcol_cur, const unsigned* vcol_next,
                               unsigned* ucol_next, uint8_t* vtq_next, cudaStream_t st) {
    LaunchScope ls(P, KK_PACK_V, st);
    k_descend_fixup_cols<<<grid_for(P, P.r * 256, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.nkbN, P.rowsVT, vcol_cur,
                                                                        vcol_next, ucol_next, vtq_next, P.d_scal,
                                                                        P.d_opt);
}

void launch_descend_fixup(Plan& P, const float* V, const unsigned* vrow_cur, unsigned* vrow_next,
                          const unsigned* urow_cur, unsigned* urow_next, const unsigned* vcol_cur, unsigned* vcol_next,
                          cudaStream_t st) {
    LaunchScope ls(P, KK_PACK_V, st);
    k_descend_fixup<<<grid_for(P, P.rowsV * 256, 256), 256, 0, st>>>(
        V, P.idx->N, P.r, P.rowsV, P.nkbV, P.rowsVT, vrow_cur, vrow_next, urow_cur, urow_next, vcol_cur, vcol_next,
        P.d_vq, P.d_scal, P.d_opt);
}

}  // namespace sos

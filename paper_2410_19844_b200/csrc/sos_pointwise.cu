// sos_pointwise.cu -- HBM-bound kernels of the step: operand split/pack of V
// and of the residual matrix R, and the fused residual + loss reduction (the
// optimiser update of PAPER.md:221 runs inside the backward GEMM, sos_gemm2.cu).  All are coalesced, vectorised where the
// layout allows, and sized as a multiple of the SM count (grid-stride).
#include <cuda_fp16.h>

#include "sos_internal.cuh"
#include "sos_split.cuh"

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

// ---------------------------------------------------------------- absmax ---
__global__ void k_absmax(const float* __restrict__ x, int64_t len, unsigned int* __restrict__ out) {
    float m = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const int64_t n4 = len >> 2;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        for (int64_t t = tid; t < n4; t += stride) {
            float4 v = __ldg(x4 + t);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
        for (int64_t t = (n4 << 2) + tid; t < len; t += stride) m = fmaxf(m, fabsf(x[t]));
    } else {
        for (int64_t t = tid; t < len; t += stride) m = fmaxf(m, fabsf(x[t]));
    }
    m = warp_max(m);
    __shared__ float s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = (threadIdx.x < (blockDim.x >> 5)) ? s[threadIdx.x] : 0.f;
        m = warp_max(m);
        if (threadIdx.x == 0) atomicMax(out, __float_as_uint(m));
    }
}

// --------------------------------------------------------------- pack V ----
// One block = 32 rows (j) x 64 columns (c) of V.  Writes the VS tile rows
// (K = column) and the VTS tile rows (K = row) of the S-layout.
__global__ void __launch_bounds__(256) k_pack_v(const float* __restrict__ V, int64_t N, int64_t r, int64_t Np,
                                                int64_t rK, int64_t rN, Scalars* __restrict__ sc,
                                                uint8_t* __restrict__ VS, uint8_t* __restrict__ VTS) {
    __shared__ float tile[32][65];
    const int tid = threadIdx.x;
    const int64_t j0 = (int64_t)blockIdx.y * 32;
    const int64_t c0 = (int64_t)blockIdx.x * 64;
    const float s = split_scale(sc->absmax_v);
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) sc->s_v = s;
    for (int e = tid; e < 32 * 64; e += 256) {
        const int jj = e >> 6, cc = e & 63;
        const int64_t j = j0 + jj, c = c0 + cc;
        tile[jj][cc] = (j < N && c < r) ? V[j * r + c] * s : 0.f;
    }
    __syncthreads();
    {  // VS: 32 rows x 2 K-blocks x 4 chunks
        const int jj = tid >> 3, h = (tid >> 2) & 1, q = tid & 3;
        const int64_t kb = (c0 >> 5) + h;
        if (kb < (rK >> 5)) {
            float x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = tile[jj][h * 32 + q * 8 + t];
            const int64_t row = j0 + jj;
            store_split_row(VS + (kb * Np + row) * 128, row, q, x);
        }
    }
    {  // VTS: 64 rows (c) x 4 chunks, K-block jb = j0/32
        const int cc = tid >> 2, q = tid & 3;
        const int64_t c = c0 + cc;
        if (c < rN) {
            float x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = tile[q * 8 + t][cc];
            store_split_row(VTS + ((j0 >> 5) * rN + c) * 128, c, q, x);
        }
    }
}

// ------------------------------------------------------------- pack VS ----
// VS only: thread (row i, K-block kb, chunk q) splits V[i][32kb+8q .. +8].
// A warp reads 256 consecutive floats of one row and writes 8 full 128-byte
// S-layout rows.
__global__ void __launch_bounds__(256) k_pack_vs(const float* __restrict__ V, int64_t N, int64_t r, int64_t Np,
                                                 int64_t nkb, Scalars* __restrict__ sc, uint8_t* __restrict__ VS) {
    const float s = split_scale(sc->absmax_v);
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->s_v = s;
    const int64_t total = Np * nkb * 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int q = (int)(t & 3);
        const int64_t rest = t >> 2;
        const int64_t i = rest / nkb, kb = rest - i * nkb;
        const int64_t c0 = kb * 32 + q * 8;
        float x[8];
        if (i < N && c0 + 8 <= r) {
            const float* src = V + i * r + c0;
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = __ldg(src + e) * s;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (i < N && c0 + e < r) ? __ldg(V + i * r + c0 + e) * s : 0.f;
        }
        store_split_row(VS + (kb * Np + i) * 128, i, q, x);
    }
}

// ------------------------------------------------------------- residual ----
// res = coef - p ; loss += res^2 ; pnorm2 += p^2 ; absmax_r = max |res|
__global__ void k_residual(const float* __restrict__ coef, const float* __restrict__ p, float* __restrict__ res,
                           int64_t M, Scalars* __restrict__ sc) {
    double l = 0.0, pn = 0.0;
    float m = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += stride) {
        const float pv = p[t];
        const float rv = coef[t] - pv;
        res[t] = rv;
        l += (double)rv * rv;
        pn += (double)pv * pv;
        m = fmaxf(m, fabsf(rv));
    }
    l = warp_sum(l);
    pn = warp_sum(pn);
    m = warp_max(m);
    __shared__ double s_l[32], s_p[32];
    __shared__ float s_m[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_l[w] = l; s_p[w] = pn; s_m[w] = m; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        l = lane < nw ? s_l[lane] : 0.0;
        pn = lane < nw ? s_p[lane] : 0.0;
        m = lane < nw ? s_m[lane] : 0.f;
        l = warp_sum(l);
        pn = warp_sum(pn);
        m = warp_max(m);
        if (lane == 0) {
            atomicAdd(&sc->loss, l);
            atomicAdd(&sc->pnorm2, pn);
            atomicMax(&sc->absmax_r, __float_as_uint(m));
        }
    }
}

// --------------------------------------------------------------- pack R ----
// R_ij = res[rank(alpha_i + alpha_j)] gathered through the pair-rank table,
// written as the RS S-layout (same [jb][i][32] row structure as PT).
__global__ void __launch_bounds__(256) k_pack_r(const uint32_t* __restrict__ pt, const float* __restrict__ res,
                                                int64_t rows8, Scalars* __restrict__ sc, uint8_t* __restrict__ RS,
                                                double stop_tol) {
    if (descent_stopped(sc, stop_tol)) return;
    const float s = split_scale(sc->absmax_r);
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->s_r = s;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows8; t += stride) {
        const uint4* p4 = reinterpret_cast<const uint4*>(pt + t * 8);
        const uint4 k0 = __ldg(p4), k1 = __ldg(p4 + 1);
        const uint32_t k[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = (k[e] != kInvalidRank) ? __ldg(res + k[e]) * s : 0.f;
        const int64_t row = t >> 2;  // = jb*Np + i ; i & 7 == row & 7 since Np % 8 == 0
        store_split_row(RS + row * 128, row, (int)(t & 3), x);
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

void launch_absmax_v(Plan& P, const float* V, cudaStream_t st) {
    const int64_t len = P.idx->N * P.r;
    LaunchScope ls(P, KK_ABSMAX_V, st);
    k_absmax<<<grid_for(P, len / 4, 256), 256, 0, st>>>(V, len, &P.d_scal->absmax_v);
}

void launch_absmax_res(Plan& P, const float* res, cudaStream_t st) {
    LaunchScope ls(P, KK_ABSMAX_R, st);
    k_absmax<<<grid_for(P, P.idx->M / 4, 256), 256, 0, st>>>(res, P.idx->M, &P.d_scal->absmax_r);
}

void launch_pack_v(Plan& P, const float* V, bool with_vts, cudaStream_t st) {
    LaunchScope ls(P, KK_PACK_V, st);
    if (with_vts) {
        dim3 grid((unsigned)(P.rN / 64), (unsigned)(P.idx->Np / 32));
        k_pack_v<<<grid, 256, 0, st>>>(V, P.idx->N, P.r, P.idx->Np, P.rK, P.rN, P.d_scal, P.d_vs, P.d_vts);
    } else {
        const int64_t work = P.idx->Np * (P.rK / 32) * 4;
        k_pack_vs<<<grid_for(P, work, 256), 256, 0, st>>>(V, P.idx->N, P.r, P.idx->Np, P.rK / 32, P.d_scal, P.d_vs);
    }
}

void launch_residual(Plan& P, const float* coef, const float* p, float* res, cudaStream_t st) {
    LaunchScope ls(P, KK_RESIDUAL, st);
    k_residual<<<grid_for(P, P.idx->M, 256, 4), 256, 0, st>>>(coef, p, res, P.idx->M, P.d_scal);
}

void launch_pack_r(Plan& P, const float* res, cudaStream_t st, double stop_tol) {
    const int64_t rows8 = P.idx->Np * P.idx->Np / 8;
    LaunchScope ls(P, KK_PACK_R, st);
    k_pack_r<<<grid_for(P, rows8, 256), 256, 0, st>>>(P.idx->d_pt, res, rows8, P.d_scal, P.d_rs, stop_tol);
}

}  // namespace sos

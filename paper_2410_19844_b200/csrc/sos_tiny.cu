// sos_tiny.cu -- the whole descent of a SMALL problem in one cooperative kernel
// (Plan::tiny, DESIGN.md 5.2 "tiny plans").
//
// For N, r of a few hundred the split step's four launches (two tcgen05 GEMMs,
// k_mid, the update) are latency-bound: ~34 us per step at config 1 (N = r =
// 330) for ~55 M multiply-adds.  Here one persistent cooperative kernel runs
// all K steps of sos_descend; a step is four grid-synchronised phases over
// fp32 CUDA-core tiles (32 x 32 outputs, K staged 32 wide in shared memory):
//   F  forward   G_ij = sum_k V_ik V_jk on the upper 32-block triangle, each
//                G_ij (weight 2 above the diagonal, 1 on it) added straight to
//                coef[rank(alpha_i + alpha_j)];
//                t += 1 (Adam) by one thread
//   L  residual  res = coef - p, loss and |p|^2 (fp64, per-block partials),
//                coef cleared for the next step
//   B  backward  every block sums the partials in the same order; unless the
//                stopping rule holds, grad += 4 R V (gradient of Eq. 2) with R
//                gathered through PT tile by tile, into a zeroed gradient buffer
//   U  update    GD / Adam, elementwise; the gradient buffer
//                cleared.  (U only after every block's B: B reads all of V.)
// The work items of F and B are (tile, K-slice) pairs -- a few K-chunks each,
// so that ~all resident blocks have one: a block walks its slice's chunks one
// after another (each waits for its loads), so parallel slices, not deeper
// per-block loops, hide the latency.  F's partial Gram tiles go straight into
// coef (the scatter is linear), B's into the gradient buffer (red.add).
// fp32 FMA accumulation over K <= a few hundred is fp32-class (~1e-7 relative,
// like the int8-slice tensor-core path); no slices, no maxima, no V^T copy.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sm100_ptx.cuh"
#include "sos_internal.cuh"

namespace sos {

constexpr int kT = 32;             // output tile edge and K chunk
constexpr int kTinyThreads = 256;  // thread = column tx = t & 31, rows ty + 8q (q < 4), ty = t >> 5

struct TinyArgs {
    float* V;
    float* m;
    float* v;
    const float* p;
    float* coef;
    float* res;
    const uint32_t* pt;
    int64_t N, r, M;
    int adam;
    DevOpt* opt;
    Scalars* sc;
    float* grad;   // N x r, zero between steps
    double* part;  // [gridDim][2]
    int64_t steps;
    int nbN, nbR;  // 32-blocks of rows / of r
    int chF, chB;  // K-chunks per work item of F (over r) and of B (over N)
    int trace;     // experiment build: block 0 prints the phase times of step 10
};
#ifdef SOS_EXPERIMENTS
#define TINY_MARK(k) do { if (a.trace && step == 10 && blockIdx.x == 0 && t == 0) { \
    unsigned long long now_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_)); tm[k] = now_; } } while (0)
#else
#define TINY_MARK(k) do { } while (0)
#endif

__device__ __forceinline__ double tiny_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double tiny_block_sum(double x, double* red, int t) {
    x = tiny_warp_sum(x);
    if ((t & 31) == 0) red[t >> 5] = x;
    __syncthreads();
    double s = 0.0;
    if (t < 32) {
        s = t < kTinyThreads / 32 ? red[t] : 0.0;
        s = tiny_warp_sum(s);
    }
    __syncthreads();  // red reused
    return s;         // valid in thread 0
}

__global__ void __launch_bounds__(kTinyThreads, 4) k_tiny_descend(const TinyArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ float As[kT][kT + 1];
    __shared__ float Bs[kT][kT + 1];
    __shared__ double red[kTinyThreads / 32];
    __shared__ double tot_s[2];
    const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
    const int64_t gtid = blockIdx.x * (int64_t)kTinyThreads + t, gstride = (int64_t)gridDim.x * kTinyThreads;
    const int64_t N = a.N, r = a.r;
    const int64_t nfwd = (int64_t)a.nbN * (a.nbN + 1) / 2, nbwd = (int64_t)a.nbN * a.nbR;
    const double tol = a.opt->stop_tol;
#ifdef SOS_EXPERIMENTS
    unsigned long long tm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
    for (int64_t step = 0; step < a.steps; ++step) {
        TINY_MARK(0);
        // ---- F: Gram tiles {I <= J} scattered into coef
        if (blockIdx.x == 0 && t == 0) advance_step(a.opt);  // read by U, after three barriers
        const int64_t sF = (a.nbR + a.chF - 1) / a.chF;  // K-slices per Gram tile
        for (int64_t w = blockIdx.x; w < nfwd * sF; w += gridDim.x) {
            const int64_t f = w / sF, k_lo = (w % sF) * a.chF * kT, k_hi = min(r, k_lo + (int64_t)a.chF * kT);
            int64_t J = (int64_t)((sqrt(8.0 * (double)f + 1.0) - 1.0) * 0.5);
            while (J * (J + 1) / 2 > f) --J;
            while ((J + 1) * (J + 2) / 2 <= f) ++J;
            const int64_t I = f - J * (J + 1) / 2;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            for (int64_t k0 = k_lo; k0 < k_hi; k0 += kT) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = t + kTinyThreads * u, row = e >> 5, kk = e & 31;
                    const int64_t i = I * kT + row, j = J * kT + row, k = k0 + kk;
                    As[row][kk] = i < N && k < r ? a.V[i * r + k] : 0.f;
                    Bs[row][kk] = j < N && k < r ? a.V[j * r + k] : 0.f;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < kT; ++kk) {
                    const float b = Bs[tx][kk];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = fmaf(As[ty + 8 * q][kk], b, acc[q]);
                }
                __syncthreads();
            }
            const int64_t j = J * kT + tx;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t i = I * kT + ty + 8 * q;
                if (i < N && j < N && i <= j) {
                    const uint32_t rk = __ldg(a.pt + pt_entry(i, j));
                    red_add_f32(a.coef + rk, (i < j ? 2.f : 1.f) * acc[q]);
                }
            }
        }
        TINY_MARK(1);
        grid.sync();
        TINY_MARK(2);
        // ---- L: residual, loss, |p|^2; coef cleared for the next step (each
        // coefficient is read and cleared by the same thread)
        {
            double l = 0.0, pn = 0.0;
            for (int64_t e = gtid; e < a.M; e += gstride) {
                const float pv = __ldg(a.p + e);
                const float rv = a.coef[e] - pv;
                a.coef[e] = 0.f;
                a.res[e] = rv;
                l += (double)rv * rv;
                pn += (double)pv * pv;
            }
            l = tiny_block_sum(l, red, t);
            pn = tiny_block_sum(pn, red, t);
            if (t == 0) {
                a.part[2 * blockIdx.x] = l;
                a.part[2 * blockIdx.x + 1] = pn;
            }
        }
        TINY_MARK(3);
        grid.sync();
        TINY_MARK(4);
        // ---- B: totals (same order in every block), stopping rule, grad tiles
        {
            double l = 0.0, pn = 0.0;
            for (int b = t; b < (int)gridDim.x; b += kTinyThreads) {
                l += a.part[2 * b];
                pn += a.part[2 * b + 1];
            }
            l = tiny_block_sum(l, red, t);
            pn = tiny_block_sum(pn, red, t);
            if (t == 0) {
                tot_s[0] = l;
                tot_s[1] = pn;
            }
            __syncthreads();
        }
        const bool stopped = tol > 0.0 && tot_s[0] <= tol * tot_s[1];
        if (blockIdx.x == gridDim.x - 1 && t == 0) {  // the step's records
            a.sc->loss = tot_s[0];
            a.sc->pnorm2 = tot_s[1];
            double* L = a.opt->losses;
            if (L) L[a.opt->loss_idx++] = tot_s[0];
        }
        if (stopped) continue;  // grid-uniform: the next step's F (coef is clear)

        const int64_t sB = (a.nbN + a.chB - 1) / a.chB;  // K-slices per gradient tile
        for (int64_t w = blockIdx.x; w < nbwd * sB; w += gridDim.x) {
            const int64_t b = w / sB, j_lo = (w % sB) * a.chB * kT, j_hi = min(N, j_lo + (int64_t)a.chB * kT);
            const int64_t I = b / a.nbR, C = b % a.nbR;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            for (int64_t j0 = j_lo; j0 < j_hi; j0 += kT) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = t + kTinyThreads * u, row = e >> 5, kk = e & 31;
                    // A: R[i][j0 + kk] through PT (res is written in this kernel: plain loads)
                    const int64_t i = I * kT + row, j = j0 + kk;
                    float rv = 0.f;
                    if (i < N && j < N) {
                        const uint32_t rk = __ldg(a.pt + pt_entry_sym(i, j));
                        rv = a.res[rk];
                    }
                    As[row][kk] = rv;
                    // B: V[j0 + row][C * 32 + kk], stored transposed (Bs[col][j])
                    const int64_t jj = j0 + row, c = C * kT + kk;
                    Bs[kk][row] = jj < N && c < r ? a.V[jj * r + c] : 0.f;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < kT; ++kk) {
                    const float bv = Bs[tx][kk];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = fmaf(As[ty + 8 * q][kk], bv, acc[q]);
                }
                __syncthreads();
            }
            const int64_t c = C * kT + tx;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t i = I * kT + ty + 8 * q;
                if (i < N && c < r) red_add_f32(a.grad + i * r + c, 4.f * acc[q]);
            }
        }
        TINY_MARK(5);
        grid.sync();  // every block has read V; the gradient is complete
        TINY_MARK(6);
        // ---- U: the update (elementwise), gradient buffer cleared
        {
            const DevOpt o = *a.opt;
            for (int64_t e = gtid; e < N * r; e += gstride) {
                const float gv = a.grad[e];
                a.grad[e] = 0.f;
                if (a.adam) {
                    float mm = a.m[e], vv = a.v[e];
                    mm = o.b1 * mm + (1.f - o.b1) * gv;
                    vv = o.b2 * vv + (1.f - o.b2) * gv * gv;
                    a.m[e] = mm;
                    a.v[e] = vv;
                    a.V[e] -= o.lr_c1 * mm / (sqrtf(vv) * o.inv_sqrt_c2 + o.eps);
                } else {
                    a.V[e] -= o.lr * gv;
                }
            }
        }
        TINY_MARK(7);
        grid.sync();  // V_{t+1} complete before the next F
        TINY_MARK(8);
#ifdef SOS_EXPERIMENTS
        if (a.trace && step == 10 && blockIdx.x == 0 && t == 0)
            printf("k_tiny step (us): F %.2f | sync %.2f | L %.2f | sync %.2f | B %.2f | sync %.2f | U %.2f | sync %.2f "
                   "(grid %d, chF %d, chB %d)\n", (tm[1] - tm[0]) * 1e-3, (tm[2] - tm[1]) * 1e-3, (tm[3] - tm[2]) * 1e-3,
                   (tm[4] - tm[3]) * 1e-3, (tm[5] - tm[4]) * 1e-3, (tm[6] - tm[5]) * 1e-3, (tm[7] - tm[6]) * 1e-3,
                   (tm[8] - tm[7]) * 1e-3, (int)gridDim.x, a.chF, a.chB);
#endif
    }
}

// blocks of the cooperative grid: all that fit at once
int tiny_grid_for(int num_sms) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tiny_descend, kTinyThreads, 0) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        return 0;
    }
    return num_sms * nb;
}

int launch_tiny_descend(Plan& P, float* V, const float* p, int64_t steps, cudaStream_t st) {
    LaunchScope ls(P, KK_TINY, st);
    TinyArgs a;
    a.V = V;
    a.m = P.d_m;
    a.v = P.d_v;
    a.p = p;
    a.coef = P.d_coef;
    a.res = P.d_res;
    a.pt = P.idx->d_pt;
    a.N = P.idx->N;
    a.r = P.r;
    a.M = P.idx->M;
    a.adam = P.opt_kind == 1 ? 1 : 0;
    a.opt = P.d_opt;
    a.sc = P.d_scal;
    a.grad = P.d_grad;
    a.part = P.d_part;
    a.steps = steps;
    a.nbN = (int)((a.N + kT - 1) / kT);
    a.nbR = (int)((a.r + kT - 1) / kT);
    // K-chunks per work item: the fewest that give no more items than blocks
    const int64_t G = P.tiny_grid, nf = (int64_t)a.nbN * (a.nbN + 1) / 2, nbw = (int64_t)a.nbN * a.nbR;
    a.chF = (int)std::max<int64_t>(1, (nf * a.nbR + G - 1) / G);
    a.chB = (int)std::max<int64_t>(1, (nbw * a.nbN + G - 1) / G);
    a.trace = 0;
    unsigned grid = (unsigned)P.tiny_grid;
#ifdef SOS_EXPERIMENTS
    {
        const char* e = getenv("SOS_TINY_TRACE");
        a.trace = e && atoi(e) ? 1 : 0;
        const char* g = getenv("SOS_TINY_GRID");  // blocks per SM (<= the occupancy limit)
        if (g && atoi(g) > 0) grid = std::min<unsigned>(grid, (unsigned)(atoi(g) * P.num_sms));
        const char* c = getenv("SOS_TINY_CH");  // "F,B" chunks per work item
        if (c) sscanf(c, "%d,%d", &a.chF, &a.chB);
    }
#endif
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);

    cfg.blockDim = dim3(kTinyThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_tiny_descend, a) == cudaSuccess ? 0 : -1;
}

}  // namespace sos

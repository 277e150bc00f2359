// sos_index.cu -- monomial index on the device (combinatorial number system).
//
// m_d = the C(n+d-1, d) degree-d monomials; the target form
// has C(n+2d-1, 2d) coefficients.  A degree-D monomial is identified with the
// sorted multiset m_1 <= ... <= m_D of its variable indices; its rank is
//     rank = sum_{k=1..D} C(m_k + k - 1, k)
// (combinatorial number system on c_k = m_k + k - 1, strictly increasing),
// which is colex order and reproduces the paper's (x1^2, x1x2, x2^2).
// The rank of a product alpha_i + alpha_j is the rank of the merged multiset.
#include <algorithm>

#include "sos_internal.cuh"

namespace sos {

// colex unranking of a degree-D multiset over n variables
__device__ __forceinline__ void unrank_colex(uint32_t rank, int D, int n, const uint32_t* binom, int bstride,
                                             uint8_t* ms) {
    uint32_t rem = rank;
    for (int k = D; k >= 1; --k) {
        int c = n + k - 2;  // largest admissible c_k
        while (c >= k && binom[c * bstride + k] > rem) --c;
        if (c < k) c = k - 1;  // C(k-1, k) = 0
        rem -= (c >= k) ? binom[c * bstride + k] : 0u;
        ms[k - 1] = (uint8_t)(c - (k - 1));
    }
}

__global__ void k_unrank_alpha(int64_t N, int d, int n, const uint32_t* __restrict__ g_binom, int nb,
                               uint8_t* __restrict__ ms_out, uint8_t* __restrict__ alpha_out) {
    extern __shared__ uint32_t s_binom[];
    const int bstride = 2 * d + 1;
    for (int t = threadIdx.x; t < nb * bstride; t += blockDim.x) s_binom[t] = g_binom[t];
    __syncthreads();
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    uint8_t ms[kMaxDeg2];
    unrank_colex((uint32_t)t, d, n, s_binom, bstride, ms);
    for (int k = 0; k < d; ++k) ms_out[t * d + k] = ms[k];
    for (int v = 0; v < n; ++v) alpha_out[t * n + v] = 0;
    for (int k = 0; k < d; ++k) alpha_out[t * n + ms[k]] += 1;
}

__global__ void k_unrank_beta(int64_t M, int D, int n, const uint32_t* __restrict__ g_binom, int nb,
                              uint8_t* __restrict__ beta_out) {
    extern __shared__ uint32_t s_binom[];
    const int bstride = D + 1;
    for (int t = threadIdx.x; t < nb * bstride; t += blockDim.x) s_binom[t] = g_binom[t];
    __syncthreads();
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= M) return;
    uint8_t ms[kMaxDeg2];
    unrank_colex((uint32_t)t, D, n, s_binom, bstride, ms);
    uint8_t ex[kMaxVars];
    for (int v = 0; v < n; ++v) ex[v] = 0;
    for (int k = 0; k < D; ++k) ex[ms[k]] += 1;
    for (int v = 0; v < n; ++v) beta_out[t * n + v] = ex[v];
}

// rank(alpha_i + alpha_j): merge the two sorted d-multisets, sum C(m'_k + k - 1, k)
__device__ __forceinline__ uint32_t pair_rank(const uint8_t* mi, const uint8_t* mj, int d, const uint32_t* binom,
                                              int bstride) {
    int a = 0, b = 0;
    uint32_t rank = 0;
    for (int k = 1; k <= 2 * d; ++k) {
        int v;
        if (b >= d || (a < d && mi[a] <= mj[b])) v = mi[a++];
        else v = mj[b++];
        rank += binom[(v + k - 1) * bstride + k];
    }
    return rank;
}

// PT, one block triangle (pt_entry in sos_internal.cuh); one thread per entry
__global__ void k_pair_table(int64_t N, int64_t Np, int d, const uint32_t* __restrict__ g_binom, int nb,
                             const uint8_t* __restrict__ ms, uint32_t* __restrict__ pt) {
    extern __shared__ uint32_t s_binom[];
    const int bstride = 2 * d + 1;
    for (int t = threadIdx.x; t < nb * bstride; t += blockDim.x) s_binom[t] = g_binom[t];
    __syncthreads();
    const int64_t total = pt_entries(Np);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // row r of the layout = 64 J (J+1) / 2 + i: block column J, then row i < 64 (J+1)
        const int64_t r = t >> 6, q = r >> 6;  // q: row in units of 64-row groups
        int64_t jb = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
        while (jb * (jb + 1) / 2 > q) --jb;
        while ((jb + 1) * (jb + 2) / 2 <= q) ++jb;
        const int64_t i = r - jb * (jb + 1) / 2 * 64;
        const int64_t j = jb * kPtW + (t & 63);
        uint32_t out = kInvalidRank;
        if (i < N && j < N) {
            uint8_t mi[kMaxDeg2 / 2], mj[kMaxDeg2 / 2];
            for (int k = 0; k < d; ++k) {
                mi[k] = ms[i * d + k];
                mj[k] = ms[j * d + k];
            }
            out = pair_rank(mi, mj, d, s_binom, bstride);
        }
        pt[t] = out;
    }
}

__global__ void k_pair_lookup(const uint32_t* __restrict__ pt, int64_t N, int64_t Np, const int64_t* __restrict__ I,
                              const int64_t* __restrict__ J, int64_t cnt, uint32_t* __restrict__ out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    int64_t i = I[t], j = J[t];
    uint32_t v = kInvalidRank;
    if (i >= 0 && j >= 0 && i < N && j < N) v = pt[pt_entry_sym(i, j)];
    out[t] = v;
}

// ---------------------------------------------- R row maxima by lattice DP --
// rrow[i] = max_j |res[rank(alpha_i + alpha_j)]| = the maximum of |res| over
// all degree-2d monomials divisible by x^alpha_i.  Computed downward through the
// monomial lattice instead of gathering the N^2 entries of R:
//     L_2d(beta) = |res_beta|,   L_D(mu) = max_v L_{D+1}(mu + e_v)   (deg mu = D)
// so L_d(alpha_i) = rrow[i].  Level D costs C(n+D-1, D) * n lookups (for
// n = 17, 2d = 10: ~50 M, against N^2 = 414 M gathers).  For mu (sorted
// multiset m_0 <= ... <= m_{D-1}) the rank of mu + e_v inserts v at position p:
//     rank = sum_{q<p} C(m_q + q, q+1) + C(v + p, p+1) + sum_{q>=p} C(m_q + q+1, q+2).
__global__ void k_rmax_level(int D, int n, int d, const uint32_t* __restrict__ g_binom, int nb,
                             const float* __restrict__ prev, bool prev_is_res, float* __restrict__ out,
                             unsigned* __restrict__ out_bits, int64_t count, const Scalars* sc, const DevOpt* opt,
                             int use_stop) {
    if (descent_stopped(sc, opt, use_stop)) return;
    extern __shared__ uint32_t s_binom[];
    const int bstride = 2 * d + 1;
    for (int t = threadIdx.x; t < nb * bstride; t += blockDim.x) s_binom[t] = g_binom[t];
    __syncthreads();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        uint8_t ms[kMaxDeg2];
        unrank_colex((uint32_t)t, D, n, s_binom, bstride, ms);
        // suffix sums of the shifted terms, prefix sums running below
        uint32_t suf[kMaxDeg2 + 1];
        suf[D] = 0;
        for (int q = D - 1; q >= 0; --q) suf[q] = suf[q + 1] + s_binom[(ms[q] + q + 1) * bstride + q + 2];
        uint32_t pre = 0;
        int p = 0;
        float best = 0.f;
        for (int v = 0; v < n; ++v) {
            while (p < D && ms[p] <= v) {
                pre += s_binom[(ms[p] + p) * bstride + p + 1];
                ++p;
            }
            const uint32_t rk = pre + s_binom[(v + p) * bstride + p + 1] + suf[p];
            const float x = __ldg(prev + rk);
            best = fmaxf(best, prev_is_res ? fabsf(x) : x);
        }
        if (out_bits) out_bits[t] = __float_as_uint(best);
        else out[t] = best;
    }
}

void launch_rmax_dp(const Index& ix, const float* res, float* scratch, unsigned* rrow, cudaStream_t st,
                    const Scalars* sc, const DevOpt* opt, int use_stop) {
    const int bstride = 2 * ix.d + 1;
    const size_t shm = sizeof(uint32_t) * ix.nb * bstride;
    const float* prev = res;
    bool prev_res = true;
    float* buf = scratch;
    for (int D = 2 * ix.d - 1; D >= ix.d; --D) {
        const int64_t count = rmax_level_count(ix.n, D);
        const bool last = D == ix.d;
        const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
        k_rmax_level<<<(unsigned)std::max<int64_t>(blocks, 1), 256, shm, st>>>(
            D, ix.n, ix.d, ix.d_binom, ix.nb, prev, prev_res, last ? nullptr : buf, last ? rrow : nullptr, count, sc,
            opt, use_stop);
        prev = buf;
        prev_res = false;
        buf += count;
    }
}

void launch_index_build(Index& ix, cudaStream_t st) {
    const int bstride = 2 * ix.d + 1;
    size_t shm = sizeof(uint32_t) * ix.nb * bstride;
    int64_t blocks = (ix.N + 255) / 256;
    k_unrank_alpha<<<(unsigned)blocks, 256, shm, st>>>(ix.N, ix.d, ix.n, ix.d_binom, ix.nb, ix.d_ms, ix.d_alpha);
    k_pair_table<<<148 * 8, 256, shm, st>>>(ix.N, ix.Np, ix.d, ix.d_binom, ix.nb, ix.d_ms, ix.d_pt);
}

void launch_beta_table(const Index& ix, uint8_t* beta, cudaStream_t st) {
    const int bstride = 2 * ix.d + 1;
    size_t shm = sizeof(uint32_t) * ix.nb * bstride;
    int64_t blocks = (ix.M + 255) / 256;
    k_unrank_beta<<<(unsigned)blocks, 256, shm, st>>>(ix.M, 2 * ix.d, ix.n, ix.d_binom, ix.nb, beta);
}

void launch_pair_lookup(const Index& ix, const int64_t* i, const int64_t* j, int64_t cnt, uint32_t* out,
                        cudaStream_t st) {
    if (cnt <= 0) return;
    k_pair_lookup<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(ix.d_pt, ix.N, ix.Np, i, j, cnt, out);
}

}  // namespace sos

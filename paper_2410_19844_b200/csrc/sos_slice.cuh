// sos_slice.cuh -- the three-slice int8 representation of fp32 operand rows
// (see sos_internal.cuh): with c = 127 / max|row| and x = value * c (|x| <= 127),
//     a1 = rint(x),  a2 = rint(254 (x - a1)),  a3 = rint(254 (254 (x - a1) - a2)),
// so x = a1 + a2/254 + a3/254^2 + e with |e| <= 0.5/254^2 and |a_s| <= 127.
#pragma once
#include <cstdint>

namespace sos {

// 127 / max for a row maximum given as float bits (0 for an all-zero row)
__device__ __forceinline__ float slice_scale(unsigned max_bits) {
    const float m = __uint_as_float(max_bits);
    return m > 0.f ? 127.f / m : 0.f;
}
// u = max / 127: the factor that turns slice products back into values
__device__ __forceinline__ float slice_unit(unsigned max_bits) { return __uint_as_float(max_bits) * (1.f / 127.f); }

__device__ __forceinline__ void slice1(float x, int& a1, int& a2, int& a3) {
    const float t1 = fminf(fmaxf(rintf(x), -127.f), 127.f);
    const float y = (x - t1) * 254.f;  // x - t1 exact; |y| <= 127
    const float t2 = rintf(y);
    const float t3 = rintf((y - t2) * 254.f);  // y - t2 exact
    a1 = (int)t1;
    a2 = (int)t2;
    a3 = (int)t3;
}

// 16 consecutive K-values of one row (scaled by c inside) -> one 16-byte chunk per slice
__device__ __forceinline__ void slice16(const float* v, float c, uint4 (&q)[3]) {
    uint32_t w[3][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int a1, a2, a3;
            slice1(v[4 * g + e] * c, a1, a2, a3);
            b0 |= (uint32_t)(a1 & 0xFF) << (8 * e);
            b1 |= (uint32_t)(a2 & 0xFF) << (8 * e);
            b2 |= (uint32_t)(a3 & 0xFF) << (8 * e);
        }
        w[0][g] = b0;
        w[1][g] = b1;
        w[2][g] = b2;
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) q[s] = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

// byte offset of chunk c (16 K-values) of row `row`, K-block kb, slice s in a Q-layout
__device__ __forceinline__ int64_t q_offset(int s, int64_t kb, int64_t row, int c, int64_t nkb, int64_t rows_total) {
    return ((s * nkb + kb) * rows_total + row) * 64 + ((c ^ (int)((row >> 1) & 3)) << 4);
}

__device__ __forceinline__ void store_q16(uint8_t* base, int64_t kb, int64_t row, int c, int64_t nkb,
                                          int64_t rows_total, const uint4 (&q)[3]) {
#pragma unroll
    for (int s = 0; s < 3; ++s) *reinterpret_cast<uint4*>(base + q_offset(s, kb, row, c, nkb, rows_total)) = q[s];
}

// VTQ row k (a column of V), K = j (a row of V): a 64 (j) x 64 (k) tile of V is
// transposed through shared memory; thread (k, chunk c) writes 16 j's.  Used by
// k_pack_vtq and by the aux warps of the forward GEMM (barrier id 1).
__device__ __forceinline__ void pack_vtq_tile(const float* __restrict__ V, int64_t N, int64_t r, int64_t rowsVT,
                                              int64_t nkbN, const unsigned* __restrict__ vcol,
                                              uint8_t* __restrict__ VTQ, int64_t jb, int64_t k0,
                                              float (*tile)[65], int t, int nthreads) {
    const int64_t j0 = jb * 64;
    for (int e = t; e < 64 * 64; e += nthreads) {
        const int jj = e >> 6, kk = e & 63;
        const int64_t j = j0 + jj, k = k0 + kk;
        tile[jj][kk] = (j < N && k < r) ? __ldg(V + j * r + k) : 0.f;
    }
    if (nthreads == 256) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"r"(nthreads));
    for (int e = t; e < 64 * 4; e += nthreads) {
        const int kk = e >> 2, c = e & 3;
        const int64_t k = k0 + kk;
        if (k >= rowsVT) continue;
        const float sc = k < r ? slice_scale(__ldg(vcol + k)) : 0.f;
        float x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = tile[c * 16 + u][kk];
        uint4 q[3];
        slice16(x, sc, q);
        store_q16(VTQ, jb, k, c, nkbN, rowsVT, q);
    }
    if (nthreads == 256) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"r"(nthreads));
}

}  // namespace sos

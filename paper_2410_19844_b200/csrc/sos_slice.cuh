// sos_slice.cuh -- the three-slice int8 representation of fp32 operand rows
// (see sos_internal.cuh).  With c = 127 * 2^16 / max|row| and the fixed-point
// value q = rint(value * c) (|q| <= 127 * 2^16 + 1), the balanced base-256
// digits of q are the slices:
//     a3 = int8(q mod 256),  q2 = (q + 128) >> 8,
//     a2 = int8(q2 mod 256), a1 = (q2 + 128) >> 8,
// so q = a1 * 2^16 + a2 * 2^8 + a3 exactly, a1 in [-127, 127], a2, a3 in
// [-128, 127], and value = (max / 127) (a1 + a2 / 256 + a3 / 65536) up to
// the rounding of q (<= 2^-16 in units of max / 127, i.e. 6e-8 of the row max).
#pragma once
#include <cstdint>

namespace sos {

// 127 * 2^16 / max for a row maximum given as float bits (0 for an all-zero row)
__device__ __forceinline__ float slice_scale(unsigned max_bits) {
    const float m = __uint_as_float(max_bits);
    return m > 0.f ? 8323072.f / m : 0.f;
}
// u = max / 127: the factor that turns slice products back into values
__device__ __forceinline__ float slice_unit(unsigned max_bits) { return __uint_as_float(max_bits) * (1.f / 127.f); }

// 16 consecutive K-values of one row -> one 16-byte chunk per slice
__device__ __forceinline__ void slice16(const float* v, float c, uint4 (&q)[3]) {
    uint32_t w[3][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        int d3[4], d2[4], d1[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int x = __float2int_rn(v[4 * g + e] * c);
            const int x2 = (x + 128) >> 8;
            d3[e] = x;                 // low byte = a3
            d2[e] = x2;                // low byte = a2
            d1[e] = (x2 + 128) >> 8;   // a1
        }
        // gather the low bytes of four ints into one word
        w[2][g] = __byte_perm(__byte_perm(d3[0], d3[1], 0x0040), __byte_perm(d3[2], d3[3], 0x0040), 0x5410);
        w[1][g] = __byte_perm(__byte_perm(d2[0], d2[1], 0x0040), __byte_perm(d2[2], d2[3], 0x0040), 0x5410);
        w[0][g] = __byte_perm(__byte_perm(d1[0], d1[1], 0x0040), __byte_perm(d1[2], d1[3], 0x0040), 0x5410);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) q[s] = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

// 4 consecutive K-values of one row -> one 4-byte word per slice (the same digits
// as slice16; word w of a 16-byte chunk holds K-values 4w .. 4w+3)
__device__ __forceinline__ void slice4(const float* v, float c, uint32_t (&q)[3]) {
    int d3[4], d2[4], d1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int x = __float2int_rn(v[e] * c);
        const int x2 = (x + 128) >> 8;
        d3[e] = x;
        d2[e] = x2;
        d1[e] = (x2 + 128) >> 8;
    }
    q[2] = __byte_perm(__byte_perm(d3[0], d3[1], 0x0040), __byte_perm(d3[2], d3[3], 0x0040), 0x5410);
    q[1] = __byte_perm(__byte_perm(d2[0], d2[1], 0x0040), __byte_perm(d2[2], d2[3], 0x0040), 0x5410);
    q[0] = __byte_perm(__byte_perm(d1[0], d1[1], 0x0040), __byte_perm(d1[2], d1[3], 0x0040), 0x5410);
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

// A 64 x 64 fp32 tile of R in shared memory (16 KB, no padding), its 16-byte
// slots XOR-swizzled so that the access patterns of the R packers are free of
// bank conflicts with 256 threads:
//   * the gather of PT block ranks, two thread maps (kGather):
//       kGatherRows: thread t stores slot (t & 15) of row 16u + (t >> 4) (a
//         quarter-warp: one row x 8 consecutive slots) -- k_mid;
//       kGatherBlocks (rt_gather_pos): a quarter-warp stores rows {2m, 2m+1} x 4
//         consecutive slots -- k_pack_rq_sym, k_rmax;
//   * rt_row16: thread (r = t >> 2, c = t & 3) loads row r, columns 16c .. 16c+15
//     as four float4 (a quarter-warp: rows {2m, 2m+1} x c = 0..3);
//   * rt_at column reads: thread (r, c) reads row 16c + e, column r (a warp:
//     rows 16c + e for c = 0..3 x 8 consecutive columns).
// slot = col4 ^ g(row) ^ 2 (col4 >> 3): the col4 term separates c from c + 2 in
// a row read; rows 2m and 2m+1 differ in bit 0 of g (row reads) and, for
// kGatherBlocks, also in bit 2 (its gather); bits 1-2 of g take 4 distinct values
// on rows 16c + e, c = 0..3 (column reads).
enum { kGatherRows = 0, kGatherBlocks = 1 };
template <int kGather>
__device__ __forceinline__ int rt_slot(int row, int col4) {
    const int g = kGather == kGatherBlocks
                      ? (row & 1) | (((row >> 4) & 1) << 1) | ((((row >> 5) ^ row) & 1) << 2)
                      : (row & 1) | (((row >> 4) & 3) << 1);
    return col4 ^ g ^ (((col4 >> 3) & 1) << 1);
}
// kGatherBlocks' thread -> (row, 4-column group) map: iteration u (0..3) of warp w
// covers rows 8 (b >> 2) .. +7 x column groups 4 (b & 3) .. +3, b = 8u + w, so one
// warp-wide gather touches 8 rows x 4 columns (stride 4).  Pair ranks of nearby
// rows and columns share or neighbour their product monomials: ~11 distinct
// 32-byte sectors of res per 32 gathers at config 4 against ~18.7 for 2 rows x 16
// column groups (tools/gather_sectors.py); the PT loads stay 64-byte row segments.
__device__ __forceinline__ void rt_gather_pos(int t, int u, int& row, int& col4) {
    const int b = u * 8 + (t >> 5), l = t & 31;
    row = 8 * (b >> 2) + (l >> 2);
    col4 = 4 * (b & 3) + (l & 3);
}
template <int kGather>
__device__ __forceinline__ void rt_store4(float* tile, int row, int col4, float4 v) {
    reinterpret_cast<float4*>(tile + row * 64)[rt_slot<kGather>(row, col4)] = v;
}
template <int kGather>
__device__ __forceinline__ float rt_at(const float* tile, int row, int col) {
    return tile[row * 64 + rt_slot<kGather>(row, col >> 2) * 4 + (col & 3)];
}
template <int kGather>
__device__ __forceinline__ void rt_row16(const float* tile, int row, int c, float (&x)[16]) {
    const float4* p = reinterpret_cast<const float4*>(tile + row * 64);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 w = p[rt_slot<kGather>(row, 4 * c + k)];
        x[4 * k] = w.x;
        x[4 * k + 1] = w.y;
        x[4 * k + 2] = w.z;
        x[4 * k + 3] = w.w;
    }
}

// VTQ row k (a column of V), K = j (a row of V): a 64 (j) x 64 (k) tile of V is
// transposed through shared memory; thread (k, chunk c) writes 16 j's.  Used by
// k_pack_vtq, k_mid (kThreads = 256, __syncthreads) and by the aux warps of the
// forward GEMM (kThreads = 64, named barrier 1).  The tile's loads are unrolled
// so that they are all in flight together.
template <int kThreads>
__device__ __forceinline__ void pack_vtq_tile(const float* __restrict__ V, int64_t N, int64_t r, int64_t rowsVT,
                                              int64_t nkbN, const unsigned* __restrict__ vcol,
                                              uint8_t* __restrict__ VTQ, int64_t jb, int64_t k0,
                                              float (*tile)[65], int t) {
    const int64_t j0 = jb * 64;
    constexpr int kLoads = 64 * 64 / kThreads;
    float x[kLoads < 16 ? kLoads : 16];
#pragma unroll
    for (int b0 = 0; b0 < kLoads; b0 += 16) {
#pragma unroll
        for (int u = 0; u < 16 && b0 + u < kLoads; ++u) {
            const int e = t + (b0 + u) * kThreads;
            const int jj = e >> 6, kk = e & 63;
            const int64_t j = j0 + jj, k = k0 + kk;
            x[u] = (j < N && k < r) ? V[j * r + k] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 16 && b0 + u < kLoads; ++u) {
            const int e = t + (b0 + u) * kThreads;
            tile[e >> 6][e & 63] = x[u];
        }
    }
    if (kThreads == 256) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"n"(kThreads));
    for (int e = t; e < 64 * 4; e += kThreads) {
        const int kk = e >> 2, c = e & 3;
        const int64_t k = k0 + kk;
        if (k >= rowsVT) continue;
        const float sc = k < r ? slice_scale(__ldg(vcol + k)) : 0.f;
        float xs[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) xs[u] = tile[c * 16 + u][kk];
        uint4 q[3];
        slice16(xs, sc, q);
        store_q16(VTQ, jb, k, c, nkbN, rowsVT, q);
    }
    if (kThreads == 256) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"n"(kThreads));
}

}  // namespace sos

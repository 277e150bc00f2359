// sos_split.cuh -- the fp16 hi/lo split of fp32 operands into the S-layout
// (see sos_internal.cuh): x*s = hi + lo, hi = fp16(x*s), lo = fp16(x*s - hi).
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

namespace sos {

// power-of-two scale s with max|x| * s < 2^14 (fp16 hi/lo split headroom)
__device__ __forceinline__ float split_scale(unsigned int absmax_bits) {
    float a = __uint_as_float(absmax_bits);
    if (!(a > 0.f) || !isfinite(a)) return 1.f;
    int e;
    frexpf(a, &e);  // a = f * 2^e, f in [0.5, 1)  =>  a < 2^e
    return ldexpf(1.f, 14 - e);
}

// x*s = hi + lo with hi = fp16(x*s), lo = fp16(x*s - hi): ~22 significant bits
__device__ __forceinline__ void split8(const float* x, uint4& hi, uint4& lo) {
    __half h[8], l[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        h[t] = __float2half_rn(x[t]);
        l[t] = __float2half_rn(x[t] - __half2float(h[t]));
    }
    hi = *reinterpret_cast<uint4*>(h);
    lo = *reinterpret_cast<uint4*>(l);
}

// write 8 already-scaled values as chunk q of a 128-byte S-layout row
__device__ __forceinline__ void store_split_row(uint8_t* row128, int64_t row, int q, const float* x8) {
    uint4 hi, lo;
    split8(x8, hi, lo);
    const int sw = (int)(row & 7);
    reinterpret_cast<uint4*>(row128)[q ^ sw] = hi;
    reinterpret_cast<uint4*>(row128)[(4 + q) ^ sw] = lo;
}

}  // namespace sos

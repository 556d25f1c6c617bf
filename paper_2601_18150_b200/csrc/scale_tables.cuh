// scale_tables.cuh -- the quantizers' per-block / per-group scale without a division.
//
// For a BF16 amax with exponent field E and significand m = 128 + mantissa (amax = m 2^(E-134)):
//     amax / 448 = (m / 7) 2^(E-140)
// and while the results stay normal, rounding commutes with the power of two, so
//     s = RN32(amax / 448)  = RN32(m / 7) 2^(E-140)
//     r = RN32(1 / s)       = RN32(1 / RN32(m / 7)) 2^(140-E)
// i.e. two 128-entry tables (filled once per CTA with IEEE div.rn / rcp.rn) and an exponent
// add replace div.rn + rcp.rn (~60 instructions) per block or group.  Valid for E >= 23
// (amax >= 2^-104, exactly the guarded-Markstein fast path: s >= 2^-113, r <= 2^113) and
// E <= 254; every other amax keeps the division path.  The exhaustive (x, amax) GPU test
// covers every BF16 amax through both paths.
#pragma once
#include <cstdint>

namespace fp8q {

struct ScaleTables {
    float s7[128];  // RN32(m / 7),         m = 128 .. 255
    float r7[128];  // RN32(1 / RN32(m / 7))
};

__device__ __forceinline__ void init_scale_tables(ScaleTables& t) {
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        const float sm = __fdiv_rn(static_cast<float>(128 + i), 7.0f);
        t.s7[i] = sm;
        t.r7[i] = __frcp_rn(sm);
    }
}

// ab = sign-cleared BF16 bits of amax with 0x0B80 <= ab < 0x7F80.
__device__ __forceinline__ void table_scale_rcp(const ScaleTables& t, uint32_t ab, float& s, float& r) {
    const int e = static_cast<int>(ab >> 7);
    const uint32_t mi = ab & 0x7Fu;
    s = __int_as_float(__float_as_int(t.s7[mi]) + ((e - 140) << 23));
    r = __int_as_float(__float_as_int(t.r7[mi]) + ((140 - e) << 23));
}

}  // namespace fp8q

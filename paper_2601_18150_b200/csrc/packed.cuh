// packed.cuh -- packed binary32 pair arithmetic (sm_100 f32x2: FMUL2 / FFMA2 / FADD2, one
// instruction for two IEEE round-to-nearest operations) and the pair form of the guarded
// Markstein quotient shared by the quantizers (quant.cu) and the producer-fused quantizers
// (producers.cu).  Every operation is the same correctly rounded binary32 operation as its
// scalar form, element by element.
#pragma once
#include <cstdint>

namespace fp8q {

__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    return (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float lo_of(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi_of(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
// a BF16 pair word (hi:lo) -> the two values as a binary32 pair (exact)
__device__ __forceinline__ uint64_t bf16x2_to_f32x2(uint32_t w) {
    return pack2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// (x0, x1) -> (RN32(x0 / s), RN32(x1 / s)) for blocks with amax >= 2^-104 (guarded Markstein:
// q0 = x r, e = fma(-q0, s, x), q1 = fma(e, r, q0) with r = RN(1/s); see quant.cu);
// rr = (r, r), nss = (-s, -s).  The sign of a zero quotient is fixed by the caller (sign OR).
__device__ __forceinline__ uint64_t quot2_fast(uint64_t x, uint64_t rr, uint64_t nss) {
    const uint64_t q0 = mul2(x, rr);
    const uint64_t e = fma2(q0, nss, x);
    return fma2(e, rr, q0);
}
// BF16 pair from a binary32 pair, round to nearest even (first source -> high half)
__device__ __forceinline__ uint32_t f32x2_to_bf16x2(uint64_t v) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_of(v)), "f"(lo_of(v)));
    return r;
}

}  // namespace fp8q

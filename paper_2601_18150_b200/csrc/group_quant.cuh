// group_quant.cuh -- the element map of the quantizers (readings Q1-Q7) as
// device helpers shared by every kernel that writes E4M3 activations or weights: the
// quantizers (quant.cu) and the decode GEMM's fused activation quantization
// (gemm_skinny.cu), so all of them produce the same bytes by construction.
//   amax bits: max over sign-cleared BF16 bit patterns (>= 0x7F80: non-finite input);
//   s = RN32(amax / 448), amax == 0 -> 1 (division, or the table path of scale_tables.cuh);
//   code = E4M3_RNE_satfinite(RN32(x / s)), guarded Markstein quotient for amax >= 2^-104,
//   the sign of x re-imposed (-0 -> 0x80).
#pragma once
#include <cstdint>

#include "packed.cuh"
#include "ptx.cuh"

namespace fp8q {

constexpr uint32_t kAmaxFastGuardBits = 0x0B80u;  // BF16 bits of 2^-104
constexpr uint32_t kNonFiniteBits = 0x7F80u;      // |x| bits >= this: Inf or NaN

// max over the 8 sign-cleared BF16 bit patterns of a 16-byte vector
__device__ __forceinline__ uint32_t vec_abs_max_bits(const uint4& v) {
    const uint32_t m = 0x7FFF7FFFu;
    uint32_t a = __vmaxu2(__vmaxu2(v.x & m, v.y & m), __vmaxu2(v.z & m, v.w & m));
    return max(a & 0xFFFFu, a >> 16);
}

__device__ __forceinline__ float scale_from_amax_bits(uint32_t ab) {
    // amax == 0 -> 1 (reading Q5); otherwise one IEEE binary32 division (reading Q4)
    return ab == 0u ? 1.0f : __fdiv_rn(__uint_as_float(ab << 16), 448.0f);
}

// max(|a|, |b|) per BF16 lane in one HMNMX2 (.NaN: a NaN input gives the canonical NaN, so
// NaN/Inf still surface as sign-cleared bits >= 0x7F80; the result's sign is garbage and is
// masked once at the end).  For every non-NaN BF16 the float order of |x| is the integer order
// of its sign-cleared bits, so this returns the same amax bits as the integer max it replaces
// (3 ALU instructions per word pair -> 1).
__device__ __forceinline__ uint32_t bmax_abs2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t abs_max_bits16(const uint32_t (&w)[8]) {
    const uint32_t a = bmax_abs2(bmax_abs2(bmax_abs2(w[0], w[1]), bmax_abs2(w[2], w[3])),
                                 bmax_abs2(bmax_abs2(w[4], w[5]), bmax_abs2(w[6], w[7]))) &
                       0x7FFF7FFFu;
    return max(a & 0xFFFFu, a >> 16);
}
// 2 NW BF16 (NW words) -> 2 NW E4M3 codes (NW / 2 words).
// Fast path: the guarded Markstein quotient evaluated NEGATED, -q1 = fma(e, -r, -q0) with
// -q0 = x (-r) and e = fma(-q0, s, x) (the same e as fma(q0, -s, x); every step is the exact
// negation of the unnegated one, RN being sign-symmetric), then code(q1) = code(-q1) ^ 0x80.
// The negated form gets the sign of a zero quotient right by itself (x = -0: -q0 = +0, e = +0,
// -q1 = +0 -> 0x80; x = +0: -q1 = -0 -> 0x00), so the input sign bits need not be gathered.
template <bool kFast, int NW>
__device__ __forceinline__ void encode_words(const uint32_t* w, float s, float r, uint32_t* c) {
    const uint64_t nrr = pack2(-r, -r);
    const uint64_t ss = pack2(s, s);
#pragma unroll
    for (int i = 0; i < NW / 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        if (kFast) {
            const uint64_t xa = pack2(__uint_as_float(wa << 16), __uint_as_float(wa & 0xFFFF0000u));
            const uint64_t xb = pack2(__uint_as_float(wb << 16), __uint_as_float(wb & 0xFFFF0000u));
            const uint64_t na = mul2(xa, nrr), nb = mul2(xb, nrr);  // -q0
            const uint64_t ea = fma2(na, ss, xa), eb = fma2(nb, ss, xb);  // e = x - q0 s
            const uint64_t qa = fma2(ea, nrr, na), qb = fma2(eb, nrr, nb);  // -q1 = -(q0 + e r)
            c[i] = (cvt_e4m3x2(lo_of(qa), hi_of(qa)) | (cvt_e4m3x2(lo_of(qb), hi_of(qb)) << 16)) ^ 0x80808080u;
        } else {
            const float q0 = __fdiv_rn(__uint_as_float(wa << 16), s);
            const float q1 = __fdiv_rn(__uint_as_float(wa & 0xFFFF0000u), s);
            const float q2 = __fdiv_rn(__uint_as_float(wb << 16), s);
            const float q3 = __fdiv_rn(__uint_as_float(wb & 0xFFFF0000u), s);
            const uint32_t sign = __byte_perm(wa, wb, 0x7531) & 0x80808080u;  // input sign bits
            c[i] = (cvt_e4m3x2(q0, q1) | (cvt_e4m3x2(q2, q3) << 16)) | sign;
        }
    }
}
// 16 BF16 (8 words) -> 16 E4M3 codes (4 words).
template <bool kFast>
__device__ __forceinline__ uint4 encode16(const uint32_t (&w)[8], float s, float r) {
    uint32_t c[4];
    encode_words<kFast, 8>(w, s, r, c);
    return make_uint4(c[0], c[1], c[2], c[3]);
}
// 8 BF16 (4 words) -> 8 E4M3 codes (2 words), the same operations per element.
template <bool kFast>
__device__ __forceinline__ uint2 encode8w(const uint32_t (&w)[4], float s, float r) {
    uint32_t c[2];
    encode_words<kFast, 4>(w, s, r, c);
    return make_uint2(c[0], c[1]);
}

}  // namespace fp8q

// producers.cu -- SURVEY §8(f) NEXT-2: the activation quantizer fused into its producers on
// the Qwen3 rollout forward ("activation quantization is performed dynamically"):
//
//   rmsnorm_quantize     y = BF16(x / sqrt(mean(x^2) + eps) * gamma)  -> 1x128 E4M3 + scales
//                        (input of q/k/v and gate/up projections)
//   silu_mul_quantize    y = BF16(silu(gate) * up)                     -> 1x128 E4M3 + scales
//                        (input of down_proj)
//
// The unfused pipeline writes y (BF16) and re-reads it for quantization; here y never
// touches HBM unless the caller asks for it (optional y_out), saving 4 B per element of
// traffic (2 written + 2 read).  The quantization of y is exactly quantize_act_per_token_group
// applied to the BF16 y (same amax / scale / guarded-Markstein / satfinite element map).
//
// Producer arithmetic = DESIGN.md reading N2 (Qwen3's HF modules: binary32, two BF16
// roundings), bit-exact by construction:
//   RMSNorm   ms = RN32(sum x^2 / K) with the sum EXACT: lanes accumulate the (exact) binary64
//             squares; when the binary64 mean lies within its error bound of a binary32
//             rounding boundary (~2^-14 of rows) the warp recomputes the sum exactly in a
//             576-bit integer accumulator and rounds the exact quotient (exact_mean_sq);
//             r = __frsqrt_rn(__fadd_rn(ms, eps)) (IEEE); t = RN_BF16(RN32(x r));
//             y = RN_BF16(RN32(gamma t)).
//   SiLU-mul  s = RN_BF16(silu(g)) depends only on the 16 bits of g: a 65,536-entry table built
//             once per device by silu_table_kernel (binary64 exp, rounded directly to BF16;
//             the exhaustive GPU test checks every entry against the oracle's 60-digit value),
//             staged in shared memory; y = RN_BF16(RN32(s u)).
#include <cstdint>
#include <mutex>

#include "group_quant.cuh"
#include "packed.cuh"
#include "pdl.cuh"
#include "ptx.cuh"
#include "quant_kernels.h"
#include "scale_tables.cuh"

namespace fp8q {
namespace {

constexpr uint32_t kGuardBits = 0x0B80u;   // BF16 bits of 2^-104 (Markstein guard)
constexpr uint32_t kNonFinite = 0x7F80u;

__device__ __forceinline__ uint32_t absmax_bits8(const uint4& v) {
    const uint32_t m = 0x7FFF7FFFu;
    uint32_t a = __vmaxu2(__vmaxu2(v.x & m, v.y & m), __vmaxu2(v.z & m, v.w & m));
    return max(a & 0xFFFFu, a >> 16);
}
__device__ __forceinline__ float scale_of(uint32_t ab) {
    return ab == 0u ? 1.0f : __fdiv_rn(__uint_as_float(ab << 16), 448.0f);
}
// 8 BF16 (4 words) -> 8 codes (2 words): the quantizers' element map (group_quant.cuh) --
// fast path the negated pair Markstein quotient, slow path (amax < 2^-104 or non-finite) div.rn.
// The amax of this lane's half-warp group (lanes 0-15 / 16-31 hold one 128-channel group each).
__device__ __forceinline__ uint32_t group_amax(uint32_t ab) {
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) ab = max(ab, __shfl_xor_sync(0xFFFFFFFFu, ab, off));
    return ab;
}
// The group's scale (table path for the fast-path amax range, IEEE division otherwise), the
// scale store by lane 0 of the half-warp, and the encode of this lane's 8 values.
__device__ __forceinline__ uint2 quantize8(const uint4& y, uint32_t ab, int lane, float* scale_dst,
                                          int32_t* flag, const ScaleTables& tabs) {
    const bool fast = ab >= kGuardBits && ab < kNonFinite;
    float s, r = 0.0f;
    if (fast)
        table_scale_rcp(tabs, ab, s, r);
    else
        s = scale_of(ab);
    if ((lane & 15) == 0) {
        *scale_dst = s;
        if (ab >= kNonFinite && flag != nullptr) *flag = 1;
    }
    const uint32_t w[4] = {y.x, y.y, y.z, y.w};
    return fast ? encode8w<true>(w, s, r) : encode8w<false>(w, s, 0.0f);
}
__device__ __forceinline__ uint4 ld_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------------------
// RMSNorm mean of squares, exactly rounded: ms = RN32(S / K), S = sum x^2 over the BF16 row.
//
// Fast path: every lane holds the binary64 sum of its squares (each square is exact in
// binary64: 16 significant bits), the warp reduces them (xor butterfly, so all lanes hold the
// same s); relative error <= (terms per lane + 6) u64.  RN32(s / K) is then the correct
// rounding unless s / K lies within that error of a binary32 rounding boundary (or outside the
// binary32 normal range): there the warp takes exact_mean_sq.
//
// exact_mean_sq: S * 2^266 is an integer (x^2 = m^2 2^(2e), m <= 255, 2e >= -266) of < 534
// bits: each lane adds its squares into an 18-word accumulator, the warp sums the accumulators
// with carries, and the exact quotient S / K is rounded to nearest even by integer long
// division (remainder = sticky bit).
constexpr int kSqWords = 18;
__device__ __forceinline__ void acc_add_sq(uint32_t (&acc)[kSqWords], uint32_t b) {
    b &= 0x7FFFu;
    if (b == 0u) return;
    const uint32_t E = b >> 7;
    const uint32_t m = E ? ((b & 0x7Fu) | 0x80u) : (b & 0x7Fu);
    const uint32_t pos = E ? 2u * E - 2u : 0u;  // 2 e + 266 with e = E - 134 (E = 0: e = -133)
    const uint64_t v = static_cast<uint64_t>(m * m) << (pos & 31u);
    uint32_t w = pos >> 5;
    uint64_t cur = static_cast<uint64_t>(acc[w]) + static_cast<uint32_t>(v);
    acc[w] = static_cast<uint32_t>(cur);
    cur = (cur >> 32) + acc[w + 1] + static_cast<uint32_t>(v >> 32);
    acc[w + 1] = static_cast<uint32_t>(cur);
    for (w += 2; (cur >> 32) != 0 && w < kSqWords; ++w) {
        cur = static_cast<uint64_t>(acc[w]) + 1u;
        acc[w] = static_cast<uint32_t>(cur);
    }
}
__device__ __noinline__ float exact_mean_sq(const uint16_t* __restrict__ xrow, int k) {
    const int lane = threadIdx.x & 31;
    uint32_t acc[kSqWords];
#pragma unroll
    for (int i = 0; i < kSqWords; ++i) acc[i] = 0u;
    for (int j = lane; j < k; j += 32) acc_add_sq(acc, xrow[j]);
    for (int off = 16; off >= 1; off >>= 1) {  // butterfly: every lane ends with the total
        uint64_t carry = 0;
#pragma unroll
        for (int i = 0; i < kSqWords; ++i) {
            const uint64_t cur = carry + acc[i] + __shfl_xor_sync(0xFFFFFFFFu, acc[i], off);
            acc[i] = static_cast<uint32_t>(cur);
            carry = cur >> 32;
        }
    }
    // N = S 2^266 2^64 (two zero words below: the quotient keeps >= 51 bits for any S > 0)
    constexpr int NW = kSqWords + 2;
    uint32_t q[NW];
    uint64_t rem = 0;
    const uint32_t kk = static_cast<uint32_t>(k);
    for (int i = NW - 1; i >= 0; --i) {
        const uint64_t cur = (rem << 32) | (i >= 2 ? acc[i - 2] : 0u);
        q[i] = static_cast<uint32_t>(cur / kk);
        rem = cur - static_cast<uint64_t>(q[i]) * kk;
    }
    int top = -1;  // most significant set bit of the quotient
    for (int i = NW - 1; i >= 0 && top < 0; --i)
        if (q[i] != 0u) top = 32 * i + 31 - __clz(q[i]);
    if (top < 0) return 0.0f;  // S == 0
    // value = (Q + rem / K) 2^e0; keep 24 bits (or fewer: binary32 subnormal quantum 2^-149)
    constexpr int e0 = -266 - 64;
    const int lsb = max(top - 23, -149 - e0);
    auto bit = [&](int p) -> uint32_t { return p < 0 ? 0u : (q[p >> 5] >> (p & 31)) & 1u; };
    uint32_t kept = 0;
    for (int p = lsb + 23; p >= lsb; --p) kept = (kept << 1) | bit(p);
    bool sticky = rem != 0;
    for (int p = lsb - 2; p >= 0 && !sticky; --p) sticky = bit(p) != 0u;
    if (bit(lsb - 1) && (sticky || (kept & 1u))) ++kept;
    int ex = lsb + e0;  // value = kept 2^ex
    if (kept == (1u << 24)) {
        kept >>= 1;
        ++ex;
    }
    if (kept < (1u << 23)) return __uint_as_float(kept);  // subnormal (ex == -149)
    const int E = ex + 150;
    if (E >= 255) return __uint_as_float(0x7F800000u);
    return __uint_as_float((static_cast<uint32_t>(E) << 23) | (kept - (1u << 23)));
}
// s: the warp's binary64 sum of squares (identical in every lane); terms: squares per lane.
__device__ __forceinline__ float mean_sq_rn(double s, int k, int terms, const uint16_t* __restrict__ xrow) {
    if (!(s < 1.0e300)) return static_cast<float>(s);  // non-finite input: flagged downstream
    const double q = __ddiv_rn(s, static_cast<double>(k));
    if (q == 0.0) return 0.0f;
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(q));
    const int E64 = static_cast<int>((b >> 52) & 0x7FF);
    bool amb = true;
    if (E64 >= 1023 - 126 && E64 <= 1023 + 126) {  // binary32 normal, away from overflow
        const int64_t L = static_cast<int64_t>(b & ((1ull << 29) - 1));
        const int64_t d = L - (1ll << 28);  // distance to the binary32 midpoint, in ulp64
        amb = (d < 0 ? -d : d) <= 2 * (terms + 8);
    }
    if (!amb) return __double2float_rn(q);
    return exact_mean_sq(xrow, k);
}

// RMSNorm + quantize: one warp per token row (persistent over rows).  Pass 1 streams the row
// (HBM) and accumulates the binary64 sum of squares; pass 2 re-reads it (L2 hit: the row was
// read a moment ago), normalises, rounds to BF16 and quantizes.  Vector t of lane l covers
// channels 256 t + 8 l .. +7, i.e. group 2t + (l >= 16).  NV > 0: k = 256 NV (every Qwen3
// hidden size), compile-time trip counts; NV == 0: any k % 128 == 0 (lane predicates).
// (Measured alternative: keeping the row in registers between the passes instead of
// re-reading it from L2 halves the occupancy and is 20 % slower.)
template <int NV>
__global__ void __launch_bounds__(256, 3) rmsnorm_quantize_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ gamma, float eps, int64_t m, int64_t k_rt,
    int64_t ld_x, uint8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales, int64_t ld_s,
    uint16_t* __restrict__ y_out, int64_t ld_y, int32_t* __restrict__ flag) {
    const int k = NV > 0 ? NV * 256 : static_cast<int>(k_rt);
    const int T = NV > 0 ? NV : (k + 255) / 256;
    constexpr int P1 = NV > 0 && NV < 8 ? NV : 8;  // pass-1 loads in flight per lane
    constexpr int U2 = NV > 0 && NV < 4 ? NV : 4;  // pass-2 vectors (x and gamma) loaded before use
    __shared__ ScaleTables tabs;
    pdl_launch_dependents();
    init_scale_tables(tabs);
    __syncthreads();
    pdl_wait();  // x is the previous kernel's output (pdl.cuh)
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * 8;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); row < m; row += warps) {
        const uint16_t* xrow = x + row * ld_x;
        const uint16_t* xr = xrow + lane * 8;
        // pass 1: binary64 sum of squares (two accumulators per lane)
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 1
        for (int t0 = 0; t0 < T; t0 += P1) {
            uint4 v[P1];
#pragma unroll
            for (int u = 0; u < P1; ++u) {
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if ((NV > 0 && NV % P1 == 0) || (t0 + u < T && (t0 + u) * 256 + lane * 8 < k))
                    v[u] = *reinterpret_cast<const uint4*>(xr + (t0 + u) * 256);
            }
#pragma unroll
            for (int u = 0; u < P1; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
                    s0 = fma(lo, lo, s0);
                    s1 = fma(hi, hi, s1);
                }
            }
        }
        double s = s0 + s1;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
        const float ms = mean_sq_rn(s, k, 8 * T, xrow);
        const float r = __frsqrt_rn(__fadd_rn(ms, eps));
        const uint64_t r2 = pack2(r, r);
#pragma unroll 1
        for (int t0 = 0; t0 < T; t0 += U2) {
            uint4 xv[U2], gv[U2];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int col = (t0 + u) * 256 + lane * 8;
                xv[u] = gv[u] = make_uint4(0u, 0u, 0u, 0u);
                if ((NV > 0 && NV % U2 == 0) || (t0 + u < T && col < k)) {
                    xv[u] = *reinterpret_cast<const uint4*>(xr + (t0 + u) * 256);
                    gv[u] = __ldg(reinterpret_cast<const uint4*>(gamma + col));
                }
            }
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int t = t0 + u;
                if (t >= T) break;  // warp-uniform
                const int col = t * 256 + lane * 8;
                const bool half_live = (t * 256 + (lane >> 4) * 128) < k;  // uniform per half
                const uint32_t w[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
                const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // t = RN_BF16(RN32(x r)); y = RN_BF16(RN32(gamma t))
                    const uint32_t tb = f32x2_to_bf16x2(mul2(bf16x2_to_f32x2(w[i]), r2));
                    o[i] = f32x2_to_bf16x2(mul2(bf16x2_to_f32x2(tb), bf16x2_to_f32x2(gw[i])));
                }
                const uint4 y = make_uint4(o[0], o[1], o[2], o[3]);  // zeros past k (x and gamma were 0)
                if (y_out != nullptr && col < k) st_v4(y_out + row * ld_y + col, y.x, y.y, y.z, y.w);
                // the whole warp reduces (lanes of a dead half contribute zeros and store nothing)
                const uint32_t ab = group_amax(absmax_bits8(y));
                if (half_live) {
                    const int g = t * 2 + (lane >> 4);
                    const uint2 c = quantize8(y, ab, lane, scales + g * ld_s + row, flag, tabs);
                    st_stream_v2(q + row * ld_q + col, c.x, c.y);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// SiLU table: g_silu_tab[b] = RN_BF16(silu(g)) for the BF16 bit pattern b of g (NaN for
// non-finite g).  Built once per device (binary64: exp <= 1 ulp, one division, then a direct
// binary64 -> BF16 rounding; tests/test_gpu_producers.py checks all 65,536 entries against the
// oracle's correctly rounded values).
__device__ uint16_t g_silu_tab[1 << 16];

// binary64 -> BF16 bits, round to nearest even, one rounding.
__device__ __forceinline__ uint32_t f64_to_bf16_rn(double v) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
    const uint32_t sign = static_cast<uint32_t>(u >> 48) & 0x8000u;
    const double a = fabs(v);
    if (a < 1.1754943508222875e-38) {  // BF16 subnormal range: quantum 2^-133 (a 2^133 is exact)
        return sign | static_cast<uint32_t>(rint(a * 1.0889035741470030e40));
    }
    const uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
    const uint64_t r = (mag + 0xFFFFFFFFFFFull + ((mag >> 45) & 1u)) >> 45;  // [E64 | 7 fraction bits]
    const uint64_t bits = r - (896ull << 7);                                  // rebias 1023 -> 127
    return sign | static_cast<uint32_t>(bits >= 0x7F80u ? 0x7F80u : bits);
}
__global__ void __launch_bounds__(256) silu_table_kernel() {
    const uint32_t b = blockIdx.x * 256u + threadIdx.x;
    uint32_t out;
    if (((b >> 7) & 0xFFu) == 0xFFu) {
        out = 0x7FC0u;
    } else {
        const double g = __uint_as_float(b << 16);
        if (g == 0.0 || g > 200.0) {
            out = b;  // silu(+-0) = +-0; g > 200: g (1 - e^-g) with e^-g < 1e-86 rounds to g
        } else if (g < -200.0) {
            out = 0x8000u;  // |silu| < 200 e^-200, below half the smallest BF16 subnormal
        } else if (fabs(g) < 0x1p-30) {
            // silu(g) = g/2 + g^2/4 + O(g^4): relative to g/2 the perturbation is below 2^-31,
            // invisible to binary64 but it decides exact BF16 ties.  g/2 is exact; below 2^-126
            // (BF16 subnormal quantum 2^-133) it can be an odd multiple of 2^-134, a tie that
            // the positive g^2/4 breaks towards +infinity.
            const double h = 0.5 * g;
            const double t = fabs(h) * 0x1p133;  // exact
            if (fabs(h) < 0x1p-126 && t - floor(t) == 0.5) {
                const uint32_t mag = static_cast<uint32_t>(g > 0.0 ? ceil(t) : floor(t));
                out = (g < 0.0 ? 0x8000u : 0u) | mag;
            } else {
                out = f64_to_bf16_rn(h);
            }
        } else {
            out = f64_to_bf16_rn(g / (1.0 + exp(-g)));
        }
    }
    g_silu_tab[b] = static_cast<uint16_t>(out);
}

// SiLU(gate) * up + quantize: persistent CTAs of 16 warps; the table is staged into shared
// memory (128 KB) once per CTA; a warp item = (token row, chunk of 8 output groups); vector j of
// lane l covers outputs chunk*1024 + 256 j + 8 l .. +7 (group 2j + (l >= 16)).
constexpr int SILU_THREADS = 512;
constexpr size_t SILU_SMEM = (size_t(1) << 17);
template <bool FULL>
__global__ void __launch_bounds__(SILU_THREADS, 1) silu_mul_quantize_kernel(
    const uint16_t* __restrict__ gu, int64_t m, int64_t inter, int64_t ld_gu, uint8_t* __restrict__ q,
    int64_t ld_q, float* __restrict__ scales, int64_t ld_s, uint16_t* __restrict__ y_out, int64_t ld_y,
    int64_t chunks, int32_t* __restrict__ flag) {
    extern __shared__ __align__(16) uint16_t stab[];
    __shared__ ScaleTables tabs;
    pdl_launch_dependents();
    pdl_wait();  // gate_up (and, on a first call, the table build) come from preceding kernels
    {
        const uint4* src = reinterpret_cast<const uint4*>(g_silu_tab);
        uint4* dst = reinterpret_cast<uint4*>(stab);
        for (int i = threadIdx.x; i < (1 << 16) / 8; i += SILU_THREADS) dst[i] = src[i];
    }
    init_scale_tables(tabs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int groups = static_cast<int>(inter >> 7);
    const int64_t items = m * chunks;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (SILU_THREADS / 32);
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * (SILU_THREADS / 32) + (threadIdx.x >> 5); item < items;
         item += nwarps) {
        const int64_t row = item / chunks;
        const int chunk = static_cast<int>(item - row * chunks);
        const uint16_t* gr = gu + row * ld_gu + (lane & 15) * 8;
        uint4 gv[4], uv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int g = chunk * 8 + 2 * j + (lane >> 4);
            gv[j] = uv[j] = make_uint4(0u, 0u, 0u, 0u);
            if (FULL || g < groups) {
                gv[j] = ld_nc(gr + g * 128);
                uv[j] = ld_nc(gr + inter + g * 128);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int g = chunk * 8 + 2 * j + (lane >> 4);
            const uint32_t gw[4] = {gv[j].x, gv[j].y, gv[j].z, gv[j].w};
            const uint32_t uw[4] = {uv[j].x, uv[j].y, uv[j].z, uv[j].w};
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // y = RN_BF16(RN32(s u)), s = table[g]
                const uint32_t sb = static_cast<uint32_t>(stab[gw[i] & 0xFFFFu]) |
                                    (static_cast<uint32_t>(stab[gw[i] >> 16]) << 16);
                o[i] = f32x2_to_bf16x2(mul2(bf16x2_to_f32x2(sb), bf16x2_to_f32x2(uw[i])));
            }
            const uint4 y = make_uint4(o[0], o[1], o[2], o[3]);
            const uint32_t ab = group_amax(absmax_bits8(y));
            if (FULL || g < groups) {
                const int col = g * 128 + (lane & 15) * 8;
                if (y_out != nullptr) st_v4(y_out + row * ld_y + col, y.x, y.y, y.z, y.w);
                const uint2 c = quantize8(y, ab, lane, scales + int64_t(g) * ld_s + row, flag, tabs);
                st_stream_v2(q + row * ld_q + col, c.x, c.y);
            }
        }
    }
}

int sms() {
    static int v = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    return v;
}

}  // namespace

cudaError_t launch_rmsnorm_quantize(const uint16_t* x, const uint16_t* gamma, float eps, int64_t m, int64_t k,
                                    int64_t ld_x, uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                    uint16_t* y, int64_t ld_y, int32_t* flag, cudaStream_t stream) {
    if (m == 0 || k == 0) return cudaSuccess;
    const int64_t rows_blocks = (m + 7) / 8;
    const int64_t cap = 3LL * sms();
    const unsigned grid = static_cast<unsigned>(rows_blocks < cap ? rows_blocks : cap);
    if (k % 256 == 0 && k <= 4096) {
        switch (k / 256) {
#define RMS_FIXED(NV)                                                                                   \
    case NV:                                                                                            \
        return launch_pdl(rmsnorm_quantize_kernel<NV>, grid, 256, 0, stream, x, gamma, eps, m, k, ld_x, q, \
                          ld_q, scales, ld_s, y, ld_y, flag);
            RMS_FIXED(1) RMS_FIXED(2) RMS_FIXED(4) RMS_FIXED(8) RMS_FIXED(12) RMS_FIXED(16)
#undef RMS_FIXED
            default: break;
        }
    }
    return launch_pdl(rmsnorm_quantize_kernel<0>, grid, 256, 0, stream, x, gamma, eps, m, k, ld_x, q, ld_q, scales,
                      ld_s, y, ld_y, flag);
}

namespace {
// The SiLU table is built once per device, on the first launch's stream.  Later launches on
// other streams wait for that build (cudaStreamWaitEvent) until it has been seen complete; a
// launch inside a stream capture before then captures its own (idempotent) build.
struct SiluTableState {
    bool launched = false;
    bool complete = false;
    bool smem_attr = false;
    cudaEvent_t built = nullptr;
};
SiluTableState g_silu_state[64];
std::mutex g_silu_mu;

cudaError_t ensure_silu_table(cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_silu_mu);
    SiluTableState& st = g_silu_state[dev];
    if (!st.smem_attr) {
        e = cudaFuncSetAttribute(silu_mul_quantize_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SILU_SMEM));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(silu_mul_quantize_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(SILU_SMEM));
        if (e != cudaSuccess) return e;
        st.smem_attr = true;
    }
    if (st.complete) return cudaSuccess;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    e = cudaStreamIsCapturing(stream, &cap);
    if (e != cudaSuccess) return e;
    if (cap != cudaStreamCaptureStatusNone) {  // inside a capture: build as part of the graph
        silu_table_kernel<<<256, 256, 0, stream>>>();
        return cudaGetLastError();
    }
    if (!st.launched) {
        silu_table_kernel<<<256, 256, 0, stream>>>();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (st.built == nullptr) {
            e = cudaEventCreateWithFlags(&st.built, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        e = cudaEventRecord(st.built, stream);
        if (e != cudaSuccess) return e;
        st.launched = true;
        return cudaSuccess;
    }
    const cudaError_t qe = cudaEventQuery(st.built);
    if (qe == cudaSuccess) {
        st.complete = true;
        return cudaSuccess;
    }
    if (qe != cudaErrorNotReady) return qe;
    return cudaStreamWaitEvent(stream, st.built, 0);
}
}  // namespace

cudaError_t launch_silu_mul_quantize(const uint16_t* gu, int64_t m, int64_t inter, int64_t ld_gu, uint8_t* q,
                                     int64_t ld_q, float* scales, int64_t ld_s, uint16_t* y, int64_t ld_y,
                                     int32_t* flag, cudaStream_t stream) {
    if (m == 0 || inter == 0) return cudaSuccess;
    cudaError_t e = ensure_silu_table(stream);
    if (e != cudaSuccess) return e;
    const int64_t chunks = (inter / 128 + 7) / 8;
    const int64_t items = m * chunks;
    const int64_t per_cta = SILU_THREADS / 32;
    int64_t grid = (items + per_cta - 1) / per_cta;
    grid = grid < sms() ? grid : sms();
    if ((inter / 128) % 8 == 0)
        return launch_pdl(silu_mul_quantize_kernel<true>, static_cast<unsigned>(grid), SILU_THREADS, SILU_SMEM, stream,
                          gu, m, inter, ld_gu, q, ld_q, scales, ld_s, y, ld_y, chunks, flag);
    else
        return launch_pdl(silu_mul_quantize_kernel<false>, static_cast<unsigned>(grid), SILU_THREADS, SILU_SMEM,
                          stream, gu, m, inter, ld_gu, q, ld_q, scales, ld_s, y, ld_y, chunks, flag);
}

}  // namespace fp8q

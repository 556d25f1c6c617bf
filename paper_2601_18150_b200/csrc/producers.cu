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
// The producer arithmetic is binary32: sum of squares per lane in element order, then a
// xor-shuffle tree; inv = rsqrt_rn(mean + eps); y = RN(RN(x inv) gamma) -> BF16 RNE.
// RMSNorm makes two passes over the row (the second hits L2), so HBM sees x once.
// silu(g) = g * sigmoid(g) in an overflow-free form with approximate exp2 / reciprocal (see
// silu2(): a few binary32 ulps).  All element math runs on binary32 PAIRS (FMUL2 / FFMA2 /
// FADD2: one instruction for two correctly rounded operations, packed.cuh) -- these kernels
// are instruction-bound, not HBM-bound, with scalar math.  (The oracle evaluates the producers in
// binary64; the two BF16 results agree except for rare ties, see tests/test_gpu_producers.py.)
#include <cstdint>

#include "packed.cuh"
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
// 8 BF16 (4 words) -> 8 codes (2 words); sign bits OR-ed in (restores -0, no-op otherwise).
// Fast path: the pair Markstein quotient; slow path (amax < 2^-104 or non-finite): div.rn.
__device__ __forceinline__ uint2 encode8_fast(const uint4& v, float s, float r) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint64_t rr = pack2(r, r), nss = pack2(-s, -s);
    uint32_t c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        const uint64_t qa = quot2_fast(bf16x2_to_f32x2(wa), rr, nss);
        const uint64_t qb = quot2_fast(bf16x2_to_f32x2(wb), rr, nss);
        const uint32_t sign = __byte_perm(wa, wb, 0x7531) & 0x80808080u;
        c[i] = (cvt_e4m3x2(lo_of(qa), hi_of(qa)) | (cvt_e4m3x2(lo_of(qb), hi_of(qb)) << 16)) | sign;
    }
    return make_uint2(c[0], c[1]);
}
__device__ __noinline__ uint2 encode8_slow(const uint4& v, float s) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        const float q0 = __fdiv_rn(__uint_as_float(wa << 16), s);
        const float q1 = __fdiv_rn(__uint_as_float(wa & 0xFFFF0000u), s);
        const float q2 = __fdiv_rn(__uint_as_float(wb << 16), s);
        const float q3 = __fdiv_rn(__uint_as_float(wb & 0xFFFF0000u), s);
        const uint32_t sign = __byte_perm(wa, wb, 0x7531) & 0x80808080u;
        c[i] = (cvt_e4m3x2(q0, q1) | (cvt_e4m3x2(q2, q3) << 16)) | sign;
    }
    return make_uint2(c[0], c[1]);
}
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
    return fast ? encode8_fast(y, s, r) : encode8_slow(y, s);
}
// silu(g) = g * sigmoid(g) without overflow: with e = exp(-|g|) (never overflows),
// sigmoid = 1 / (1 + e) for g >= 0 and e / (1 + e) for g < 0.  exp via ex2.approx (no ftz:
// subnormal e stay exact enough for BF16 subnormal outputs) and rcp.approx: a few binary32
// ulps, far below the 2^-8 relative spacing of the BF16 result.
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint64_t silu2(uint64_t g2) {
    const uint64_t a2 = g2 & 0x7FFFFFFF7FFFFFFFull;  // |g|
    const uint64_t t2 = mul2(a2, pack2(-1.4426950408889634f, -1.4426950408889634f));
    const float e0 = ex2_approx(lo_of(t2)), e1 = ex2_approx(hi_of(t2));
    const uint64_t d2 = add2(pack2(e0, e1), pack2(1.0f, 1.0f));
    const float r0 = rcp_approx(lo_of(d2)), r1 = rcp_approx(hi_of(d2));
    const uint64_t er2 = mul2(pack2(e0, e1), pack2(r0, r1));
    // sigmoid: r for g >= 0, e r for g < 0 (selected by the sign bit of g)
    const float sg0 = (lo_of(g2) >= 0.0f) ? r0 : lo_of(er2);
    const float sg1 = (hi_of(g2) >= 0.0f) ? r1 : hi_of(er2);
    return mul2(g2, pack2(sg0, sg1));
}
__device__ __forceinline__ uint4 ld_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------------------
// RMSNorm + quantize: one warp per token row (persistent over rows).  Pass 1 streams the row
// (HBM) and accumulates the sum of squares; pass 2 re-reads it (L2 hit: the row was read a
// moment ago), normalises, rounds to BF16 and quantizes.  Vector t of lane l covers channels
// 256 t + 8 l .. +7, i.e. group 2t + (l >= 16).  Few registers -> many warps per SM, and
// UNROLL independent 16-byte loads per lane in flight in pass 1.
__global__ void __launch_bounds__(256, 3) rmsnorm_quantize_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ gamma, float eps, int64_t m, int64_t k,
    int64_t ld_x, uint8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales, int64_t ld_s,
    uint16_t* __restrict__ y_out, int64_t ld_y, int32_t* __restrict__ flag) {
    constexpr int UNROLL = 8;
    __shared__ ScaleTables tabs;
    init_scale_tables(tabs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * 8;
    const int T = static_cast<int>((k + 255) / 256);
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); row < m; row += warps) {
        const uint16_t* xr = x + row * ld_x + lane * 8;
        // pass 1: sum of squares, two interleaved binary32 partial sums per lane (FFMA2)
        uint64_t ss2 = 0;
        for (int t0 = 0; t0 < T; t0 += UNROLL) {
            uint4 v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if (t0 + u < T && (t0 + u) * 256 + lane * 8 < k) v[u] = *reinterpret_cast<const uint4*>(xr + (t0 + u) * 256);
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint64_t x2 = bf16x2_to_f32x2(w[i]);
                    ss2 = fma2(x2, x2, ss2);
                }
            }
        }
        float ss = __fadd_rn(lo_of(ss2), hi_of(ss2));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, off);
        const float mean = __fdiv_rn(ss, static_cast<float>(k));
        const float inv = __frsqrt_rn(__fadd_rn(mean, eps));
        const uint64_t inv2 = pack2(inv, inv);
        constexpr int U2 = 4;  // pass 2: U2 vectors of x and gamma loaded before any use
        for (int t0 = 0; t0 < T; t0 += U2) {
            uint4 xv[U2], gv[U2];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int col = (t0 + u) * 256 + lane * 8;
                xv[u] = gv[u] = make_uint4(0u, 0u, 0u, 0u);
                if (t0 + u < T && col < k) {
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
                for (int i = 0; i < 4; ++i)  // y = RN(RN(x inv) gamma), rounded to BF16
                    o[i] = f32x2_to_bf16x2(mul2(mul2(bf16x2_to_f32x2(w[i]), inv2), bf16x2_to_f32x2(gw[i])));
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

// The same computation for k = 256 NV (every Qwen3 hidden size): all loops have compile-time
// trip counts and no lane predicates (no divergence bookkeeping around the shuffles).
// (Measured alternative: keeping the row in registers between the passes instead of
// re-reading it from L2 halves the occupancy and is 20 % slower.)
template <int NV>
__global__ void __launch_bounds__(256, 3) rmsnorm_quantize_fixed_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ gamma, float eps, int64_t m, int64_t ld_x,
    uint8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scales, int64_t ld_s, uint16_t* __restrict__ y_out,
    int64_t ld_y, int32_t* __restrict__ flag) {
    constexpr int K = NV * 256;
    constexpr int P1 = NV < 8 ? NV : 8;  // pass-1 loads in flight per lane
    constexpr int U2 = NV < 4 ? NV : 4;  // pass-2 vectors (x and gamma) loaded before use
    __shared__ ScaleTables tabs;
    init_scale_tables(tabs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * 8;
    const uint16_t* gl = gamma + lane * 8;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); row < m; row += warps) {
        const uint16_t* xr = x + row * ld_x + lane * 8;
        uint8_t* qr = q + row * ld_q + lane * 8;
        uint64_t ss2 = 0;
#pragma unroll 1
        for (int t0 = 0; t0 < NV; t0 += P1) {
            uint4 v[P1];
#pragma unroll
            for (int u = 0; u < P1; ++u) v[u] = *reinterpret_cast<const uint4*>(xr + (t0 + u) * 256);
#pragma unroll
            for (int u = 0; u < P1; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint64_t x2 = bf16x2_to_f32x2(w[i]);
                    ss2 = fma2(x2, x2, ss2);
                }
            }
        }
        float ss = __fadd_rn(lo_of(ss2), hi_of(ss2));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, off);
        const float inv = __frsqrt_rn(__fadd_rn(__fdiv_rn(ss, static_cast<float>(K)), eps));
        const uint64_t inv2 = pack2(inv, inv);
#pragma unroll 1
        for (int t0 = 0; t0 < NV; t0 += U2) {
            uint4 xv[U2], gv[U2];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                xv[u] = *reinterpret_cast<const uint4*>(xr + (t0 + u) * 256);
                gv[u] = __ldg(reinterpret_cast<const uint4*>(gl + (t0 + u) * 256));
            }
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int t = t0 + u;
                const uint32_t w[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
                const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)  // y = RN(RN(x inv) gamma), rounded to BF16
                    o[i] = f32x2_to_bf16x2(mul2(mul2(bf16x2_to_f32x2(w[i]), inv2), bf16x2_to_f32x2(gw[i])));
                const uint4 y = make_uint4(o[0], o[1], o[2], o[3]);
                if (y_out != nullptr) st_v4(y_out + row * ld_y + t * 256 + lane * 8, y.x, y.y, y.z, y.w);
                const uint32_t ab = group_amax(absmax_bits8(y));
                const int g = t * 2 + (lane >> 4);
                const uint2 c = quantize8(y, ab, lane, scales + g * ld_s + row, flag, tabs);
                st_stream_v2(qr + t * 256, c.x, c.y);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// SiLU(gate) * up + quantize: one warp per (token row, chunk of 8 output groups); vector j of
// lane l covers outputs chunk*1024 + 256 j + 8 l .. +7 (group 2j + (l >= 16)).
template <bool FULL>
__global__ void __launch_bounds__(256) silu_mul_quantize_kernel(
    const uint16_t* __restrict__ gu, int64_t m, int64_t inter, int64_t ld_gu, uint8_t* __restrict__ q,
    int64_t ld_q, float* __restrict__ scales, int64_t ld_s, uint16_t* __restrict__ y_out, int64_t ld_y,
    int64_t chunks, int32_t* __restrict__ flag) {
    __shared__ ScaleTables tabs;
    init_scale_tables(tabs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (item >= m * chunks) return;
    const int64_t row = item / chunks;
    const int chunk = static_cast<int>(item - row * chunks);
    const int groups = static_cast<int>(inter >> 7);
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
        for (int i = 0; i < 4; ++i)  // y = RN(silu(g) u), rounded to BF16
            o[i] = f32x2_to_bf16x2(mul2(silu2(bf16x2_to_f32x2(gw[i])), bf16x2_to_f32x2(uw[i])));
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
#define RMS_FIXED(NV)                                                                                      \
    case NV:                                                                                               \
        rmsnorm_quantize_fixed_kernel<NV><<<grid, 256, 0, stream>>>(x, gamma, eps, m, ld_x, q, ld_q, scales, \
                                                                    ld_s, y, ld_y, flag);                  \
        return cudaGetLastError();
            RMS_FIXED(1) RMS_FIXED(2) RMS_FIXED(3) RMS_FIXED(4) RMS_FIXED(5) RMS_FIXED(6) RMS_FIXED(7)
            RMS_FIXED(8) RMS_FIXED(9) RMS_FIXED(10) RMS_FIXED(11) RMS_FIXED(12) RMS_FIXED(13) RMS_FIXED(14)
            RMS_FIXED(15) RMS_FIXED(16)
#undef RMS_FIXED
            default: break;
        }
    }
    rmsnorm_quantize_kernel<<<grid, 256, 0, stream>>>(x, gamma, eps, m, k, ld_x, q, ld_q, scales, ld_s, y, ld_y, flag);
    return cudaGetLastError();
}

cudaError_t launch_silu_mul_quantize(const uint16_t* gu, int64_t m, int64_t inter, int64_t ld_gu, uint8_t* q,
                                     int64_t ld_q, float* scales, int64_t ld_s, uint16_t* y, int64_t ld_y,
                                     int32_t* flag, cudaStream_t stream) {
    if (m == 0 || inter == 0) return cudaSuccess;
    const int64_t chunks = (inter / 128 + 7) / 8;
    const int64_t items = m * chunks;
    const int64_t blocks = (items + 7) / 8;
    if (blocks > 0x7FFFFFFFLL) return cudaErrorInvalidConfiguration;
    if ((inter / 128) % 8 == 0)
        silu_mul_quantize_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
            gu, m, inter, ld_gu, q, ld_q, scales, ld_s, y, ld_y, chunks, flag);
    else
        silu_mul_quantize_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
            gu, m, inter, ld_gu, q, ld_q, scales, ld_s, y, ld_y, chunks, flag);
    return cudaGetLastError();
}

}  // namespace fp8q

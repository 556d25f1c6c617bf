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
// silu(): a few binary32 ulps).  (The oracle evaluates the producers in
// binary64; the two BF16 results agree except for rare ties, see tests/test_gpu_producers.py.)
#include <cstdint>

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
__device__ __forceinline__ float quot(float x, float s, float r, bool fast) {
    if (!fast) return __fdiv_rn(x, s);
    const float q0 = __fmul_rn(x, r);
    const float e = __fmaf_rn(-q0, s, x);
    return __fmaf_rn(e, r, q0);
}
// 8 BF16 (4 words) -> 8 codes (2 words); sign bits OR-ed in (restores -0, no-op otherwise).
__device__ __forceinline__ uint2 encode8(const uint4& v, float s, float r, bool fast) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        const float q0 = quot(__uint_as_float(wa << 16), s, r, fast);
        const float q1 = quot(__uint_as_float(wa & 0xFFFF0000u), s, r, fast);
        const float q2 = quot(__uint_as_float(wb << 16), s, r, fast);
        const float q3 = quot(__uint_as_float(wb & 0xFFFF0000u), s, r, fast);
        const uint32_t sign = __byte_perm(wa, wb, 0x7531) & 0x80808080u;
        c[i] = (cvt_e4m3x2(q0, q1) | (cvt_e4m3x2(q2, q3) << 16)) | sign;
    }
    return make_uint2(c[0], c[1]);
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
    return encode8(y, s, r, fast);
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));  // first source -> high half
    return r;
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
__device__ __forceinline__ float silu(float g) {
    const float e = ex2_approx(-fabsf(g) * 1.4426950408889634f);
    const float r = rcp_approx(1.0f + e);
    return g >= 0.0f ? g * r : (g * e) * r;
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
        const uint16_t* xr = x + row * ld_x;
        float ss = 0.0f;
        for (int t0 = 0; t0 < T; t0 += UNROLL) {
            uint4 v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const int64_t col = int64_t(t0 + u) * 256 + lane * 8;
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if (t0 + u < T && col < k) v[u] = *reinterpret_cast<const uint4*>(xr + col);
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
                    ss = __fmaf_rn(lo, lo, ss);
                    ss = __fmaf_rn(hi, hi, ss);
                }
            }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, off);
        const float mean = __fdiv_rn(ss, static_cast<float>(k));
        const float inv = __frsqrt_rn(__fadd_rn(mean, eps));
        constexpr int U2 = 4;  // pass 2: U2 vectors of x and gamma loaded before any use
        for (int t0 = 0; t0 < T; t0 += U2) {
            uint4 xv[U2], gv[U2];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int64_t col = int64_t(t0 + u) * 256 + lane * 8;
                xv[u] = gv[u] = make_uint4(0u, 0u, 0u, 0u);
                if (t0 + u < T && col < k) {
                    xv[u] = *reinterpret_cast<const uint4*>(xr + col);
                    gv[u] = __ldg(reinterpret_cast<const uint4*>(gamma + col));
                }
            }
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int t = t0 + u;
                if (t >= T) break;  // warp-uniform
                const int64_t col = int64_t(t) * 256 + lane * 8;
                const bool half_live = (int64_t(t) * 256 + (lane >> 4) * 128) < k;  // uniform per half
                const uint32_t w[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
                const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float lo = __fmul_rn(__fmul_rn(__uint_as_float(w[i] << 16), inv), __uint_as_float(gw[i] << 16));
                    const float hi = __fmul_rn(__fmul_rn(__uint_as_float(w[i] & 0xFFFF0000u), inv),
                                               __uint_as_float(gw[i] & 0xFFFF0000u));
                    o[i] = bf16x2(lo, hi);
                }
                uint4 y = make_uint4(o[0], o[1], o[2], o[3]);  // zeros past k (x and gamma were 0)
                if (y_out != nullptr && col < k) st_v4(y_out + row * ld_y + col, y.x, y.y, y.z, y.w);
                // the whole warp reduces (lanes of a dead half contribute zeros and store nothing)
                uint32_t ab = absmax_bits8(y);
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) ab = max(ab, __shfl_xor_sync(0xFFFFFFFFu, ab, off));
                if (half_live) {
                    const int64_t g = int64_t(t) * 2 + (lane >> 4);
                    const uint2 c = quantize8(y, ab, lane, scales + g * ld_s + row, flag, tabs);
                    st_stream_v2(q + row * ld_q + col, c.x, c.y);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// SiLU(gate) * up + quantize: one warp per (token row, chunk of 8 output groups); vector j of
// lane l covers outputs chunk*1024 + 256 j + 8 l .. +7 (group 2j + (l >= 16)).
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
    const int64_t row = item / chunks, chunk = item - (item / chunks) * chunks;
    const int64_t groups = inter >> 7;
    const uint16_t* gr = gu + row * ld_gu;
    uint4 gv[4], uv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 8 + 2 * j + (lane >> 4);
        gv[j] = uv[j] = make_uint4(0u, 0u, 0u, 0u);
        if (g < groups) {
            const int64_t col = g * 128 + (lane & 15) * 8;
            gv[j] = ld_nc(gr + col);
            uv[j] = ld_nc(gr + inter + col);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 8 + 2 * j + (lane >> 4);
        const uint32_t gw[4] = {gv[j].x, gv[j].y, gv[j].z, gv[j].w};
        const uint32_t uw[4] = {uv[j].x, uv[j].y, uv[j].z, uv[j].w};
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float g0 = __uint_as_float(gw[i] << 16), g1 = __uint_as_float(gw[i] & 0xFFFF0000u);
            const float u0 = __uint_as_float(uw[i] << 16), u1 = __uint_as_float(uw[i] & 0xFFFF0000u);
            const float s0 = silu(g0);
            const float s1 = silu(g1);
            o[i] = bf16x2(__fmul_rn(s0, u0), __fmul_rn(s1, u1));
        }
        const uint4 y = make_uint4(o[0], o[1], o[2], o[3]);
        uint32_t ab = absmax_bits8(y);
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) ab = max(ab, __shfl_xor_sync(0xFFFFFFFFu, ab, off));
        if (g < groups) {
            const int64_t col = g * 128 + (lane & 15) * 8;
            if (y_out != nullptr) st_v4(y_out + row * ld_y + col, y.x, y.y, y.z, y.w);
            const uint2 c = quantize8(y, ab, lane, scales + g * ld_s + row, flag, tabs);
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
    const int64_t cap = 4LL * sms();
    const unsigned grid = static_cast<unsigned>(rows_blocks < cap ? rows_blocks : cap);
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
    silu_mul_quantize_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(gu, m, inter, ld_gu, q, ld_q, scales,
                                                                               ld_s, y, ld_y, chunks, flag);
    return cudaGetLastError();
}

}  // namespace fp8q

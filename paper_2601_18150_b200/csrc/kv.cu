// kv.cu -- SURVEY §8(f) NEXT-3: FP8 KV cache with per-step scale recalibration
// (§2.3.1; readings K1-K4 in DESIGN.md §3).
//
//   kv_amax_update      amax_bits = max(amax_bits, max |x|) over a BF16 [rows, cols] tensor, as
//                       sign-cleared BF16 bits (an integer max is exact and order-free, so the
//                       result is deterministic whatever the atomics' order); one call per
//                       calibration batch (inference side: the first forward after a sync;
//                       trainer side: every batch of the calibration subset).
//   kv_scale_from_amax  s = RN32(amax / 448), amax == 0 -> 1, for many layers at once.
//   kv_quantize_append  cache[slot[r]] = E4M3_RNE_sat(RN32(x[r] / s)) with the layer's scalar
//                       scale (read from device memory: no host sync between calibration and
//                       append) and a count of saturated elements (|RN32(x/s)| >= 464).
//
// The element map is the weights' (quant.cu): the guarded Markstein quotient on binary32 pairs
// for scales of amax >= 2^-104, div.rn below; values far beyond the calibrated range (quotient
// >= 464, including an overflowing quotient) saturate to +-448 explicitly.  HBM-bound:
// append moves 2 + 1 B per element, calibration 2 B per element.
#include <cstdint>

#include "packed.cuh"
#include "ptx.cuh"
#include "quant_kernels.h"

namespace fp8q {
namespace {

constexpr uint32_t kKvNonFinite = 0x7F80u;
// smallest scale of the Markstein fast path: RN32(2^-104 / 448) = 0x07124925 (the scale of the
// amax guard 2^-104 of quant.cu; every smaller scale takes div.rn)
__device__ __forceinline__ float kv_fast_scale_min() { return __uint_as_float(0x07124925u); }

__device__ __forceinline__ uint32_t amax_bits8(const uint4& v) {
    const uint32_t m = 0x7FFF7FFFu;
    const uint32_t a = __vmaxu2(__vmaxu2(v.x & m, v.y & m), __vmaxu2(v.z & m, v.w & m));
    return max(a & 0xFFFFu, a >> 16);
}

// ---------------------------------------------------------------- calibration (K1)
__global__ void __launch_bounds__(256) kv_amax_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t cols,
                                                      int64_t ld, int vec, uint32_t* __restrict__ amax_bits,
                                                      int32_t* __restrict__ flag) {
    uint32_t a = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // one warp per row (rows strided over the grid's warps): no per-element index division
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    (void)stride;
    (void)tid;
    if (vec) {  // 8 BF16 per lane per vector (cols % 8 == 0, 16-byte aligned rows), KU in flight
        constexpr int KU = 4;
        const int cv = static_cast<int>(cols / 8);
        for (int64_t r = w0; r < rows; r += nwarps) {
            const uint4* xr = reinterpret_cast<const uint4*>(x + r * ld);
            for (int c0 = lane; c0 < cv; c0 += 32 * KU) {
                uint4 v[KU];
#pragma unroll
                for (int u = 0; u < KU; ++u)
                    v[u] = (c0 + 32 * u < cv) ? __ldcs(xr + c0 + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int u = 0; u < KU; ++u) a = max(a, amax_bits8(v[u]));
            }
        }
    } else {
        for (int64_t r = w0; r < rows; r += nwarps)
            for (int64_t c = lane; c < cols; c += 32) a = max(a, static_cast<uint32_t>(x[r * ld + c] & 0x7FFFu));
    }
    a = __reduce_max_sync(0xFFFFFFFFu, a);
    if ((threadIdx.x & 31) == 0 && a != 0) {
        atomicMax(amax_bits, a);
        if (a >= kKvNonFinite && flag != nullptr) atomicOr(flag, 1);
    }
}

__global__ void kv_scale_kernel(const uint32_t* __restrict__ amax_bits, int64_t n, float* __restrict__ scales) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint32_t a = amax_bits[i];
        scales[i] = a == 0u ? 1.0f : __fdiv_rn(__uint_as_float(a << 16), 448.0f);
    }
}

// ---------------------------------------------------------------- append (K2-K4)
// 8 BF16 -> 8 codes with the scalar scale; returns this lane's saturated count.
template <bool kFast>
__device__ __forceinline__ uint2 kv_encode8(const uint4& v, float s, float r, uint32_t& sat) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint64_t rr = pack2(r, r), nss = pack2(-s, -s);
    uint32_t c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        float q[4];
        if (kFast) {
            const uint64_t qa = quot2_fast(bf16x2_to_f32x2(wa), rr, nss);
            const uint64_t qb = quot2_fast(bf16x2_to_f32x2(wb), rr, nss);
            q[0] = lo_of(qa), q[1] = hi_of(qa), q[2] = lo_of(qb), q[3] = hi_of(qb);
        } else {
            q[0] = __fdiv_rn(__uint_as_float(wa << 16), s);
            q[1] = __fdiv_rn(__uint_as_float(wa & 0xFFFF0000u), s);
            q[2] = __fdiv_rn(__uint_as_float(wb << 16), s);
            q[3] = __fdiv_rn(__uint_as_float(wb & 0xFFFF0000u), s);
        }
        // quotients >= 464 (incl. an overflowed or NaN Markstein quotient) saturate and count
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool o = !(fabsf(q[j]) < 464.0f);
            sat += o ? 1u : 0u;
            q[j] = o ? 448.0f : fabsf(q[j]);  // magnitude; the sign comes from the input below
        }
        const uint32_t sign = __byte_perm(wa, wb, 0x7531) & 0x80808080u;
        c[i] = (cvt_e4m3x2(q[0], q[1]) | (cvt_e4m3x2(q[2], q[3]) << 16)) | sign;
    }
    return make_uint2(c[0], c[1]);
}

__global__ void __launch_bounds__(256) kv_append_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld_x, const float* __restrict__ scale,
                                                        const int32_t* __restrict__ slots, uint8_t* __restrict__ cache,
                                                        int64_t ld_c, int64_t num_slots, int vec,
                                                        uint32_t* __restrict__ saturated, int32_t* __restrict__ flag) {
    const float s = *scale;
    const bool fast = s >= kv_fast_scale_min() && s <= 3.4e38f;
    const float r = fast ? __frcp_rn(s) : 0.0f;
    uint32_t sat = 0, bad = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // one warp per row (rows strided over the grid's warps): no per-element index division
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    (void)stride;
    (void)tid;
    if (vec) {  // KU vectors of 8 BF16 loaded per lane before any is encoded
        constexpr int KU = 4;
        const int cv = static_cast<int>(cols / 8);
        for (int64_t row = w0; row < rows; row += nwarps) {
            const int64_t dst = slots != nullptr ? slots[row] : row;
            const uint4* xr = reinterpret_cast<const uint4*>(x + row * ld_x);
            const bool ok = dst >= 0 && dst < num_slots;
            bad |= ok ? 0u : 2u;
            uint8_t* cr = cache + (ok ? dst : 0) * ld_c;
            for (int c0 = lane; c0 < cv; c0 += 32 * KU) {
                uint4 v[KU];
#pragma unroll
                for (int u = 0; u < KU; ++u)
                    v[u] = (c0 + 32 * u < cv) ? __ldcs(xr + c0 + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int u = 0; u < KU; ++u) {
                    bad |= amax_bits8(v[u]) >= kKvNonFinite ? 1u : 0u;
                    if (!ok || c0 + 32 * u >= cv) continue;
                    const uint2 code = fast ? kv_encode8<true>(v[u], s, r, sat) : kv_encode8<false>(v[u], s, r, sat);
                    st_stream_v2(cr + (c0 + 32 * u) * 8, code.x, code.y);
                }
            }
        }
    } else {
        for (int64_t row = w0; row < rows; row += nwarps) {
            const int64_t dst = slots != nullptr ? slots[row] : row;
            const bool ok = dst >= 0 && dst < num_slots;
            bad |= ok ? 0u : 2u;
            for (int64_t c = lane; c < cols; c += 32) {
                const uint16_t h = x[row * ld_x + c];
                bad |= (h & 0x7FFFu) >= kKvNonFinite ? 1u : 0u;
                if (!ok) continue;
                const float q = __fdiv_rn(__uint_as_float(static_cast<uint32_t>(h) << 16), s);
                const bool o = !(fabsf(q) < 464.0f);
                sat += o ? 1u : 0u;
                const uint32_t code = cvt_e4m3x2(o ? 448.0f : fabsf(q), 0.0f) & 0x7Fu;  // lo -> byte 0
                cache[dst * ld_c + c] = static_cast<uint8_t>(code | ((h >> 8) & 0x80u));
            }
        }
    }
    sat = __reduce_add_sync(0xFFFFFFFFu, sat);
    bad = __reduce_or_sync(0xFFFFFFFFu, bad);
    if ((threadIdx.x & 31) == 0) {
        if (sat != 0 && saturated != nullptr) atomicAdd(saturated, sat);
        if (bad != 0 && flag != nullptr) atomicOr(flag, static_cast<int32_t>(bad));
    }
}

int kv_sms() {
    static int v = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    return v;
}

unsigned kv_grid(int64_t work_items) {
    const int64_t blocks = (work_items + 255) / 256;
    const int64_t cap = 4LL * kv_sms();
    return static_cast<unsigned>(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

}  // namespace

cudaError_t launch_kv_amax(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, uint32_t* amax_bits,
                           int32_t* flag, cudaStream_t stream) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const int vec = (cols % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0) ? 1 : 0;
    kv_amax_kernel<<<kv_grid(rows * 32), 256, 0, stream>>>(x, rows, cols, ld, vec,
                                                                                     amax_bits, flag);
    return cudaGetLastError();
}

cudaError_t launch_kv_scale(const uint32_t* amax_bits, int64_t n, float* scales, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    kv_scale_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(amax_bits, n, scales);
    return cudaGetLastError();
}

cudaError_t launch_kv_append(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x, const float* scale,
                             const int32_t* slots, uint8_t* cache, int64_t ld_c, int64_t num_slots,
                             uint32_t* saturated, int32_t* flag, cudaStream_t stream) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const int vec = (cols % 8 == 0 && ld_x % 8 == 0 && ld_c % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(cache) & 7u) == 0)
                        ? 1
                        : 0;
    kv_append_kernel<<<kv_grid(rows * 32), 256, 0, stream>>>(
        x, rows, cols, ld_x, scale, slots, cache, ld_c, num_slots, vec, saturated, flag);
    return cudaGetLastError();
}

}  // namespace fp8q

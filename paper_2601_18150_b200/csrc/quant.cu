// quant.cu -- the two E4M3 quantizers of the FP8 W8A8 rollout (arXiv 2601.18150 §2.1.1).
//
//   quantize_weight_blockwise     PAPER.md:54-58, Eq. (1): one fp32 scale per 128x128 block.
//   quantize_act_per_token_group  PAPER.md:65,233: one fp32 scale per token per 128 channels.
//
// Both are HBM-bound element maps (3 B of traffic per element).  Design:
//   * 16-byte vector loads of 8 BF16, every load of a CTA issued before any use (32 KB in
//     flight per weight block, 16 KB per activation warp group) so HBM sees deep queues;
//   * amax as an INTEGER max over sign-cleared BF16 bits (__vmaxu2 on packed pairs, then a
//     redux.sync / shuffle reduction).  Widening BF16 -> fp32 is exact and order-preserving
//     on |x|, so the max of the bits is the bits of the max; bits >= 0x7F80 flag NaN/Inf;
//   * s = RN32(amax / 448) by one IEEE division per block (reading Q4), amax == 0 -> 1 (Q5);
//   * RN32(x / s) per element via the guarded Markstein sequence
//         r = RN(1/s); q0 = RN(x r); e = fma(-q0, s, x); q1 = fma(e, r, q0)
//     which gives the same E4M3 code as the IEEE quotient for every block with
//     amax >= 2^-104 (SURVEY.md §0 finding 4; re-proved on the GPU by the exhaustive
//     (x, amax) map in tests/test_gpu_exhaustive.py); the sign is re-imposed from x so that
//     x = -0 still gives -0 (IEEE: -0 / s = -0).  Blocks below the guard use div.rn;
//   * packed cvt.rn.satfinite.e4m3x2.f32 (RNE, saturating, reading Q1/Q7), 8-byte stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "ptx.cuh"
#include "quant_kernels.h"
#include "packed.cuh"
#include "scale_tables.cuh"
#include "group_quant.cuh"
#include "pdl.cuh"
#include "trace.cuh"

namespace fp8q {

namespace {


// RN32(x / s) for blocks with amax >= 2^-104 (see header comment), sign taken from x.
__device__ __forceinline__ float quot_fast(float x, float s, float r) {
    const float q0 = __fmul_rn(x, r);
    const float e = __fmaf_rn(-q0, s, x);
    const float q1 = __fmaf_rn(e, r, q0);
    return __uint_as_float((__float_as_uint(q1) & 0x7FFFFFFFu) | (__float_as_uint(x) & 0x80000000u));
}

template <bool kFast>
__device__ __forceinline__ uint2 encode8(const uint4& v, float s, float r) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float lo = __uint_as_float(w[i] << 16);
        const float hi = __uint_as_float(w[i] & 0xFFFF0000u);
        const float qlo = kFast ? quot_fast(lo, s, r) : __fdiv_rn(lo, s);
        const float qhi = kFast ? quot_fast(hi, s, r) : __fdiv_rn(hi, s);
        c[i] = cvt_e4m3x2(qlo, qhi);
    }
    return make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
}

// ---------------------------------------------------------------------------------------
// Weights: one CTA (256 threads) per 128x128 block.  Warp w covers rows 16w..16w+15; in each
// of its 8 loads, lanes 0-15 read one row's 256 B and lanes 16-31 the next row's, so every
// load instruction moves two full 256-byte row segments.
__global__ void __launch_bounds__(256) weight_blockwise_kernel(
    const uint16_t* __restrict__ w, int64_t n, int64_t k, int64_t ld_w, uint8_t* __restrict__ q,
    int64_t ld_q, float* __restrict__ scales, int64_t ld_s, int64_t nbk,
    int32_t* __restrict__ nonfinite_flag) {
    __shared__ uint32_t red[8];
    const int64_t blk = blockIdx.x;
    const int64_t bi = blk / nbk;
    const int64_t bj = blk - bi * nbk;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t col = bj * 128 + (lane & 15) * 8;
    const int64_t row0 = bi * 128 + warp * 16 + (lane >> 4);
    const bool col_ok = col < k;

    uint4 v[8];
    uint32_t ab = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = row0 + 2 * i;
        v[i] = make_uint4(0u, 0u, 0u, 0u);
        if (col_ok && row < n) v[i] = ld_stream_v4(w + row * ld_w + col);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) ab = max(ab, vec_abs_max_bits(v[i]));
    ab = __reduce_max_sync(0xFFFFFFFFu, ab);
    if (lane == 0) red[warp] = ab;
    __syncthreads();
    ab = red[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) ab = max(ab, red[i]);

    const float s = scale_from_amax_bits(ab);
    if (threadIdx.x == 0) {
        scales[bi * ld_s + bj] = s;
        if (ab >= kNonFiniteBits && nonfinite_flag != nullptr) *nonfinite_flag = 1;
    }
    if (ab >= kAmaxFastGuardBits) {
        const float r = __frcp_rn(s);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = row0 + 2 * i;
            if (col_ok && row < n) {
                const uint2 c = encode8<true>(v[i], s, r);
                st_stream_v2(q + row * ld_q + col, c.x, c.y);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = row0 + 2 * i;
            if (col_ok && row < n) {
                const uint2 c = encode8<false>(v[i], s, 0.0f);
                st_stream_v2(q + row * ld_q + col, c.x, c.y);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// Activations: one warp per (token row, chunk of 8 groups = 1024 channels).  Vector j of lane
// l covers channels chunk*1024 + j*256 + l*8, i.e. group 2j + (l >= 16): each half-warp owns
// one 128-channel group per j and reduces its amax with 4 xor-shuffles.
__global__ void __launch_bounds__(256) act_per_token_group_kernel(
    const uint16_t* __restrict__ x, int64_t m, int64_t k, int64_t ld_x, uint8_t* __restrict__ q,
    int64_t ld_q, float* __restrict__ scales, int64_t ld_s, int64_t chunks_per_row,
    int32_t* __restrict__ nonfinite_flag) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (item >= m * chunks_per_row) return;
    const int64_t row = item / chunks_per_row;
    const int64_t chunk = item - row * chunks_per_row;
    const int64_t groups = k >> 7;
    const uint16_t* xr = x + row * ld_x;

    uint4 v[4];
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 8 + 2 * j + (lane >> 4);
        ok[j] = g < groups;
        v[j] = make_uint4(0u, 0u, 0u, 0u);
        if (ok[j]) v[j] = ld_stream_v4(xr + g * 128 + (lane & 15) * 8);
    }
    uint32_t ab[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ab[j] = vec_abs_max_bits(v[j]);
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) ab[j] = max(ab[j], __shfl_xor_sync(0xFFFFFFFFu, ab[j], off));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (!ok[j]) continue;
        const int64_t g = chunk * 8 + 2 * j + (lane >> 4);
        const float s = scale_from_amax_bits(ab[j]);
        if ((lane & 15) == 0) {
            scales[g * ld_s + row] = s;
            if (ab[j] >= kNonFiniteBits && nonfinite_flag != nullptr) *nonfinite_flag = 1;
        }
        uint2 c;
        if (ab[j] >= kAmaxFastGuardBits)
            c = encode8<true>(v[j], s, __frcp_rn(s));
        else
            c = encode8<false>(v[j], s, 0.0f);
        st_stream_v2(q + row * ld_q + g * 128 + (lane & 15) * 8, c.x, c.y);
    }
}

// =======================================================================================
// Wide-vector persistent variants (the production path when alignment allows).
//   * 32-byte loads (LDG.256: 16 BF16 per thread per load) and 16-byte code stores;
//   * packed f32x2 Markstein quotient (FMUL2/FFMA2: half the instructions per element);
//   * the sign of zero is restored by OR-ing each input's sign bit into its code byte
//     (a no-op for every nonzero input, and exactly IEEE's -0 / s = -0 for x = -0);
//   * persistent CTAs/warps that issue the NEXT block's loads before encoding the current
//     one, so every SM keeps a full block of HBM reads in flight.
// =======================================================================================
__device__ __forceinline__ void ld_v8(const void* p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_v4_na(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
// ---------------------------------------------------------------------------------------
// Weights, wide path: requires k % 16 == 0, w 32-byte aligned with ld_w % 16 == 0, codes
// 16-byte aligned with ld_q % 16 == 0.  CTA = 256 threads handles whole 128x128 blocks,
// blk = blockIdx.x, += gridDim.x.  Thread (warp w, lane l) owns rows 16w + 4i + (l >> 3),
// i = 0..3, columns 16 (l & 7) .. +15 of the block: each load instruction of a warp reads
// four full 256-byte row segments.
struct WBlockRegs {
    uint32_t v[4][8];
};
struct WTensor {
    const uint16_t* w;
    uint8_t* q;
    float* scales;
    int64_t n, k, ld_w, ld_q, ld_s, nbk;
    int64_t blk0;  // first global block index of this tensor
};
struct WBatch {
    // bulk path: one 2-D tensor map per tensor (BF16 [n][k], box 128 x 128, zero OOB fill)
    CUtensorMap tm[kMaxWeightBatch];
    WTensor t[kMaxWeightBatch];
    int count;
    int64_t nblocks;
    // NEXT-1 fan-out: ndest > 0 -> every code / scale store goes to pointer + dq[d] / ds[d]
    // for each destination d (peer-mapped buffers of identical layout, e.g. symmetric
    // memory: the quantized shard lands in every rank's engine buffer, no separate gather)
    int ndest;
    int64_t dq[kMaxFanout];
    int64_t ds[kMaxFanout];
};
__device__ __forceinline__ void wq_load(const uint16_t* __restrict__ w, int64_t n, int64_t k,
                                        int64_t ld_w, int64_t nbk, int64_t blk, WBlockRegs& d) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bi = blk / nbk, bj = blk - (blk / nbk) * nbk;
    const int64_t col = bj * 128 + (lane & 7) * 16;
    const int64_t row0 = bi * 128 + warp * 16 + (lane >> 3);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = row0 + 4 * i;
        if (col < k && row < n) {
            ld_v8(w + row * ld_w + col, d.v[i]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) d.v[i][j] = 0u;
        }
    }
}
template <bool kFanout>
__device__ __forceinline__ void wq_store(uint8_t* dst, const uint4& c, const WBatch& bt) {
    if (kFanout) {
        for (int dd = 0; dd < bt.ndest; ++dd) st_v4_na(dst + bt.dq[dd], c);
    } else {
        st_v4_na(dst, c);
    }
}
template <bool kFanout>
__device__ __forceinline__ void wq_process(const WBlockRegs& d, int64_t n, int64_t k, uint8_t* __restrict__ q,
                                           int64_t ld_q, float* __restrict__ scales, int64_t ld_s,
                                           int64_t nbk, int64_t blk, uint32_t* red,
                                           int32_t* __restrict__ nonfinite_flag, const WBatch& bt,
                                           int warp = threadIdx.x >> 5, int bar_id = 0) {
    const int lane = threadIdx.x & 31;
    const int64_t bi = blk / nbk, bj = blk - (blk / nbk) * nbk;
    const int64_t col = bj * 128 + (lane & 7) * 16;
    const int64_t row0 = bi * 128 + warp * 16 + (lane >> 3);
    uint32_t ab = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) ab = max(ab, abs_max_bits16(d.v[i]));
    ab = __reduce_max_sync(0xFFFFFFFFu, ab);
    if (lane == 0) red[warp] = ab;
    if (bar_id == 0)
        __syncthreads();
    else  // the 8 warps of one consumer team (bulk kernel)
        asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory");
    ab = red[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) ab = max(ab, red[i]);
    const float s = scale_from_amax_bits(ab);
    if (warp == 0 && lane == 0) {
        if (kFanout) {
            for (int dd = 0; dd < bt.ndest; ++dd)
                *reinterpret_cast<float*>(reinterpret_cast<char*>(scales + bi * ld_s + bj) + bt.ds[dd]) = s;
        } else {
            scales[bi * ld_s + bj] = s;
        }
        if (ab >= kNonFiniteBits && nonfinite_flag != nullptr) *nonfinite_flag = 1;
    }
    const bool col_ok = col < k;
    if (ab >= kAmaxFastGuardBits) {
        const float r = __frcp_rn(s);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + 4 * i;
            if (col_ok && row < n) wq_store<kFanout>(q + row * ld_q + col, encode16<true>(d.v[i], s, r), bt);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + 4 * i;
            if (col_ok && row < n) wq_store<kFanout>(q + row * ld_q + col, encode16<false>(d.v[i], s, 0.0f), bt);
        }
    }
}
// A batch of weight tensors quantized by ONE launch (the weight sync re-quantizes every
// linear weight of a layer at once: one launch instead of one per tensor).
template <bool kFanout>
__global__ void __launch_bounds__(256, 2) weight_blockwise_wide_kernel(const __grid_constant__ WBatch bt,
                                                                        int32_t* __restrict__ nonfinite_flag) {
    __shared__ uint32_t red[2][8];
    WBlockRegs a, b;
    const int64_t nblocks = bt.nblocks;
    auto tensor_of = [&](int64_t blk) {
        int i = 0;
        while (i + 1 < bt.count && blk >= bt.t[i + 1].blk0) ++i;
        return i;
    };
    auto load = [&](int64_t blk, WBlockRegs& d) {
        const WTensor& t = bt.t[tensor_of(blk)];
        wq_load(t.w, t.n, t.k, t.ld_w, t.nbk, blk - t.blk0, d);
    };
    auto process = [&](int64_t blk, const WBlockRegs& d, uint32_t* rd) {
        const WTensor& t = bt.t[tensor_of(blk)];
        wq_process<kFanout>(d, t.n, t.k, t.q, t.ld_q, t.scales, t.ld_s, t.nbk, blk - t.blk0, rd, nonfinite_flag, bt);
    };
    int64_t blk = blockIdx.x;
    if (blk < nblocks) load(blk, a);
    while (blk < nblocks) {  // unrolled by two so the register buffers stay static
        int64_t nxt = blk + gridDim.x;
        if (nxt < nblocks) load(nxt, b);
        process(blk, a, red[0]);
        blk = nxt;
        if (blk >= nblocks) break;
        nxt = blk + gridDim.x;
        if (nxt < nblocks) load(nxt, a);
        process(blk, b, red[1]);
        blk = nxt;
    }
}

// ---------------------------------------------------------------------------------------
// Activations, wide path: requires x 32-byte aligned with ld_x % 16 == 0, codes 16-byte
// aligned with ld_q % 16 == 0.  A warp item = (token row, 16 groups = 2048 channels); vector
// j of lane l covers group 4j + (l >> 3) of the item, channels 16 (l & 7) .. +15 of it; eight
// lanes reduce a group's amax with three xor-shuffles.  Warps are persistent over items and
// prefetch their next item.
struct AItemRegs {
    uint32_t v[4][8];
};
__device__ __forceinline__ void aq_load(const uint16_t* __restrict__ x, int64_t ld_x, int64_t groups,
                                        int64_t chunks, int64_t item, AItemRegs& d) {
    const int lane = threadIdx.x & 31;
    const int64_t row = item / chunks, chunk = item - (item / chunks) * chunks;
    const uint16_t* xr = x + row * ld_x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 16 + 4 * j + (lane >> 3);
        if (g < groups) {
            ld_v8(xr + g * 128 + (lane & 7) * 16, d.v[j]);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) d.v[j][t] = 0u;
        }
    }
}
__device__ __forceinline__ void aq_process(const AItemRegs& d, uint8_t* __restrict__ q, int64_t ld_q,
                                           float* __restrict__ scales, int64_t ld_s, int64_t groups,
                                           int64_t row, int64_t chunk, int32_t* __restrict__ nonfinite_flag,
                                           const ScaleTables& tabs) {
    const int lane = threadIdx.x & 31;
    uint32_t ab[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ab[j] = abs_max_bits16(d.v[j]);
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) ab[j] = max(ab[j], __shfl_xor_sync(0xFFFFFFFFu, ab[j], off));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 16 + 4 * j + (lane >> 3);
        if (g >= groups) continue;
        const bool fast = ab[j] >= kAmaxFastGuardBits && ab[j] < kNonFiniteBits;
        float s, r = 0.0f;
        if (fast)
            table_scale_rcp(tabs, ab[j], s, r);
        else
            s = scale_from_amax_bits(ab[j]);
        if ((lane & 7) == 0) {
            scales[g * ld_s + row] = s;
            if (ab[j] >= kNonFiniteBits && nonfinite_flag != nullptr) *nonfinite_flag = 1;
        }
        uint4 c;
        if (fast)
            c = encode16<true>(d.v[j], s, r);
        else
            c = encode16<false>(d.v[j], s, 0.0f);
        st_v4_na(q + row * ld_q + g * 128 + (lane & 7) * 16, c);
    }
}
// The staged kernel's encode of one item (same arithmetic as aq_process): 32-bit indices, the
// item's row already resolved by the producer, and no divergent branches in the common case --
// when every live group of the warp is on the fast path the encode is warp-uniform; the scale
// and code stores are predicated instructions.
__device__ __forceinline__ void st_global_f32_if(bool p, float* a, float v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.global.f32 [%1], %2;\n\t}" ::"r"(
                     static_cast<uint32_t>(p)),
                 "l"(a), "f"(v)
                 : "memory");
}
__device__ __forceinline__ void st_global_v4_na_if(bool p, void* a, const uint4& v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t"
        "@q st.global.L1::no_allocate.v4.u32 [%1], {%2, %3, %4, %5};\n\t}" ::"r"(static_cast<uint32_t>(p)),
        "l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
        : "memory");
}
__device__ __forceinline__ void aq_process_item(const AItemRegs& d, uint8_t* __restrict__ qrow,
                                                float* __restrict__ srow, uint32_t ld_s, uint32_t groups,
                                                uint32_t chunk, int32_t* __restrict__ nonfinite_flag,
                                                const ScaleTables& tabs) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t ab[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ab[j] = abs_max_bits16(d.v[j]);
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) ab[j] = max(ab[j], __shfl_xor_sync(0xFFFFFFFFu, ab[j], off));
    }
    // One vote for the whole item: when every live group of the warp is on the fast path (the
    // common case) the four groups run as straight-line code, so their table loads, quotients
    // and stores interleave instead of forming four sequential vote / branch / store sections.
    bool all_fast = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool live = chunk * 16u + 4u * j + (lane >> 3) < groups;
        all_fast = all_fast && (!live || (ab[j] >= kAmaxFastGuardBits && ab[j] < kNonFiniteBits));
    }
    float s[4], r[4];
    uint4 c[4];
    if (__all_sync(0xFFFFFFFFu, all_fast)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) table_scale_rcp(tabs, ab[j], s[j], r[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = encode16<true>(d.v[j], s[j], r[j]);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool fast = ab[j] >= kAmaxFastGuardBits && ab[j] < kNonFiniteBits;
            r[j] = 0.0f;
            if (fast)
                table_scale_rcp(tabs, ab[j], s[j], r[j]);
            else
                s[j] = scale_from_amax_bits(ab[j]);
            c[j] = fast ? encode16<true>(d.v[j], s[j], r[j]) : encode16<false>(d.v[j], s[j], 0.0f);
        }
    }
    uint32_t bad = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t g = chunk * 16u + 4u * j + (lane >> 3);
        const bool live = g < groups;
        st_global_f32_if(live && (lane & 7) == 0, srow + static_cast<uint64_t>(g) * ld_s, s[j]);
        bad |= (live && ab[j] >= kNonFiniteBits) ? 1u : 0u;
        st_global_v4_na_if(live, qrow + g * 128 + (lane & 7) * 16, c[j]);
    }
    if (bad && nonfinite_flag != nullptr) *nonfinite_flag = 1;
}
__global__ void __launch_bounds__(256, 2) act_per_token_group_wide_kernel(
    const uint16_t* __restrict__ x, int64_t ld_x, uint8_t* __restrict__ q, int64_t ld_q,
    float* __restrict__ scales, int64_t ld_s, int64_t groups, int64_t chunks, int64_t items,
    int32_t* __restrict__ nonfinite_flag) {
    __shared__ ScaleTables tabs;
    const uint32_t trace_tag = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(x));
    (void)trace_tag;
    if (threadIdx.x == 0) FP8Q_TREC(trace_tag, 10);
    pdl_launch_dependents();  // the consumer GEMM may start its weight prefetch now
    init_scale_tables(tabs);
    __syncthreads();
    pdl_wait();  // x is the previous kernel's output; q / scales may still be read by it
    if (threadIdx.x == 0) FP8Q_TREC(trace_tag, 11);
    const int64_t warps = static_cast<int64_t>(gridDim.x) * 8;
    int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    AItemRegs a, b;
    if (item < items) aq_load(x, ld_x, groups, chunks, item, a);
    while (item < items) {
        int64_t nxt = item + warps;
        if (nxt < items) aq_load(x, ld_x, groups, chunks, nxt, b);
        aq_process(a, q, ld_q, scales, ld_s, groups, item / chunks, item % chunks, nonfinite_flag, tabs);
        item = nxt;
        if (item >= items) break;
        nxt = item + warps;
        if (nxt < items) aq_load(x, ld_x, groups, chunks, nxt, a);
        aq_process(b, q, ld_q, scales, ld_s, groups, item / chunks, item % chunks, nonfinite_flag, tabs);
        item = nxt;
    }
    if (threadIdx.x == 0) FP8Q_TREC(trace_tag, 12);
}

// ---------------------------------------------------------------------------------------
// Activations, bulk-staged path (production): one persistent CTA per SM owns an EQUAL
// contiguous range of units (unit = 8 token rows x 16 groups = 8 items of 2048 channels = 32 KB),
// so no SM finishes a whole item early (the warp-persistent grid above leaves a 1/7 tail at
// M = 8192, K = 4096).  A producer thread streams the range into a ring of ABQ_STAGES shared-
// memory stages, ONE unit per stage: one 3-D TMA box {128 channels, 16 groups, 8 rows} (rows
// past m and groups past the row zero-filled, completion counted in bytes on the stage's
// mbarrier) -- one copy and one barrier arrive per 32 KB, so the single issuing thread is never
// what paces the stream (with one copy per 4 KB item it was: the consumers waited on the full
// barriers 40 % of the time at 46 % issue).  Two teams of ABQ_ITEMS consumer warps take
// alternate stages; warp w encodes row w of the unit from shared memory exactly as the wide
// path does (same registers, same arithmetic) and releases the stage with one arrive.
constexpr int ABQ_ITEMS = 8;    // rows per unit = items per stage (one per warp of a team)
constexpr int ABQ_TEAMS = 2;    // consumer teams (alternate stages)
constexpr int ABQ_STAGES = 6;   // ring depth: 6 x 32 KB
constexpr int ABQ_ITEM_BYTES = 4096;
constexpr int ABQ_THREADS = (ABQ_ITEMS * ABQ_TEAMS + 1) * 32;
constexpr size_t ABQ_SMEM = size_t(ABQ_STAGES) * ABQ_ITEMS * ABQ_ITEM_BYTES + 2 * ABQ_STAGES * 8 + 128;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)),
        "l"(kL2EvictFirst)  // every byte is read exactly once
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* smem_dst, const void* desc, uint64_t* bar, int32_t c0,
                                                 int32_t c1, int32_t c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// kMasked = false: the slot's groups past the row are zeros already (the TMA box's zero fill),
// so every lane loads unconditionally.
template <bool kMasked>
__device__ __forceinline__ void aq_load_smem(uint32_t base, int64_t groups, int64_t chunk, AItemRegs& d) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t g = chunk * 16 + 4 * j + (lane >> 3);
        if (!kMasked || g < groups) {
            const uint32_t a = base + static_cast<uint32_t>((4 * j + (lane >> 3)) * 256 + (lane & 7) * 32);
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(d.v[j][0]), "=r"(d.v[j][1]), "=r"(d.v[j][2]), "=r"(d.v[j][3]) : "r"(a));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(d.v[j][4]), "=r"(d.v[j][5]), "=r"(d.v[j][6]), "=r"(d.v[j][7]) : "r"(a + 16));
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) d.v[j][t] = 0u;
        }
    }
}
// A batch of activation tensors for one launch of the staged kernel (the four GEMM inputs of a
// layer in one persistent launch: one pipeline ramp and one tail instead of four).  Units are
// numbered across the batch (tensor i owns units [unit0, unit0 + ceil(m / 8) * chunks)), row
// block major: unit = row block * chunks + chunk.
struct ATensor {
    const uint16_t* x;
    uint8_t* q;
    float* scales;
    int64_t ld_x, ld_q, ld_s, groups, m;
    int32_t chunks;  // 16-group (4 KB) items per token row
    int64_t unit0;   // first batch-global unit of this tensor
};
struct ABatch {
    CUtensorMap tm[kMaxActBatch];  // kTma: 3-D map {128 channels, groups, m}, box {128, 16, 8}
    ATensor t[kMaxActBatch];
    int count;
    int64_t units;
};
// kTma: each unit is ONE 3-D TMA box; !kTma (dev, FP8Q_ACT_LOAD=bulk): one cp.async.bulk copy
// per live row of the unit.  Same shared-memory layout (row i of the unit at 4 KB * i), same
// consumers.
template <bool kTma>
__global__ void __launch_bounds__(ABQ_THREADS, 1) act_per_token_group_bulk_kernel(
    const __grid_constant__ ABatch ab, int32_t* __restrict__ nonfinite_flag) {
    extern __shared__ __align__(128) uint8_t abq_smem[];
    __shared__ ScaleTables tabs;
    pdl_launch_dependents();
    uint64_t* full = reinterpret_cast<uint64_t*>(abq_smem + size_t(ABQ_STAGES) * ABQ_ITEMS * ABQ_ITEM_BYTES);
    uint64_t* empty = full + ABQ_STAGES;
    // per stage: {first row of the unit, tensor << 16 | chunk}, written by the producer with
    // the copy, so consumers need no division or tensor search per unit
    __shared__ uint2 meta[ABQ_STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this CTA's equal share of the batch's units
    const int64_t u0 = ab.units * blockIdx.x / gridDim.x;
    const int64_t u1 = ab.units * (blockIdx.x + 1) / gridDim.x;
    const int32_t nstages = static_cast<int32_t>(u1 - u0);
    init_scale_tables(tabs);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ABQ_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ABQ_ITEMS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // (no-op unless launched with programmatic stream serialization)
    const uint32_t ring = smem_u32(abq_smem);
    if (warp == ABQ_ITEMS * ABQ_TEAMS) {
        if (lane == 0 && nstages > 0) {
            // (tensor, row block, chunk) of the current unit, advanced incrementally
            int ti = 0;
            while (ti + 1 < ab.count && u0 >= ab.t[ti + 1].unit0) ++ti;
            int32_t chunks = ab.t[ti].chunks;
            int64_t rows = ab.t[ti].m;
            int64_t row = ((u0 - ab.t[ti].unit0) / chunks) * ABQ_ITEMS;
            int32_t chunk = static_cast<int32_t>(u0 - ab.t[ti].unit0 - (row / ABQ_ITEMS) * chunks);
            uint32_t s = 0, ph = 0;
            for (int32_t it = 0; it < nstages; ++it) {
                mbar_wait(&empty[s], ph ^ 1u);
                meta[s] = make_uint2(static_cast<uint32_t>(row),
                                     (static_cast<uint32_t>(ti) << 16) | static_cast<uint32_t>(chunk));
                if (kTma) {
                    // the whole box counts, zero-filled rows / groups included
                    mbar_arrive_expect_tx(&full[s], ABQ_ITEMS * ABQ_ITEM_BYTES);
                    tma_load_3d_hint(abq_smem + s * (ABQ_ITEMS * ABQ_ITEM_BYTES), &ab.tm[ti], &full[s], 0, chunk * 16,
                                     static_cast<int32_t>(row), kL2EvictFirst);
                } else {
                    const ATensor& t = ab.t[ti];
                    const uint32_t nb = chunk == chunks - 1
                                            ? static_cast<uint32_t>(t.groups - (chunks - 1) * 16) * 256u
                                            : 4096u;
                    const int nr = rows - row < ABQ_ITEMS ? static_cast<int>(rows - row) : ABQ_ITEMS;
                    mbar_arrive_expect_tx(&full[s], nb * static_cast<uint32_t>(nr));
                    for (int i = 0; i < nr; ++i)
                        bulk_g2s(ring + (s * ABQ_ITEMS + i) * ABQ_ITEM_BYTES, t.x + (row + i) * t.ld_x + chunk * 2048,
                                 nb, &full[s]);
                }
                if (++chunk == chunks) {
                    chunk = 0;
                    row += ABQ_ITEMS;
                    if (row >= rows && ti + 1 < ab.count) {
                        ++ti;
                        row = 0;
                        chunks = ab.t[ti].chunks;
                        rows = ab.t[ti].m;
                    }
                }
                if (++s == ABQ_STAGES) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int team = warp / ABQ_ITEMS, w = warp % ABQ_ITEMS;
    uint32_t s = static_cast<uint32_t>(team), ph = 0;
    for (int32_t it = team; it < nstages; it += ABQ_TEAMS) {
        mbar_wait(&full[s], ph);
        const uint2 md = meta[s];
        const ATensor& t = ab.t[md.y >> 16];
        const uint32_t row = md.x + static_cast<uint32_t>(w);
        if (row < static_cast<uint64_t>(t.m)) {
            const uint32_t chunk = md.y & 0xFFFFu;
            const uint32_t groups = static_cast<uint32_t>(t.groups);
            AItemRegs d;
            aq_load_smem<!kTma>(ring + (s * ABQ_ITEMS + w) * ABQ_ITEM_BYTES, groups, chunk, d);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // the row is in registers: free the slot
            aq_process_item(d, t.q + int64_t(row) * t.ld_q, t.scales + row, static_cast<uint32_t>(t.ld_s), groups,
                            chunk, nonfinite_flag, tabs);
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        s += ABQ_TEAMS;
        if (s >= ABQ_STAGES) {
            s -= ABQ_STAGES;
            ph ^= 1u;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Weights, bulk-staged path (production for the wide layout): one persistent CTA per SM owns
// an EQUAL contiguous range of the batch's 128x128 blocks (the block-strided grid above ends
// with a partial wave: 1024 blocks over 296 CTAs is 3.46 waves for o_proj).  A producer warp
// streams the range into a ring of WBQ_STAGES 32 KB shared-memory stages, one block per stage,
// with ONE 2-D TMA load per block (box 128 x 128 BF16 of the tensor's map, rows past n and
// columns past k zero-filled, completion counted in bytes on the stage's mbarrier), so up to 6
// blocks of HBM reads are in flight per SM.  (Per-row cp.async.bulk copies of 256 B were
// measured at a quarter of this rate: the copy engine is bound by requests, not bytes.)  Two teams of 8 consumer warps take alternate stages; a team reads its
// block from shared memory into exactly the registers the wide path loads from global memory,
// frees the stage, and runs the same wq_process (same arithmetic, same stores) with the block
// amax reduced over the team's named barrier.
constexpr int WBQ_STAGES = 6;
constexpr int WBQ_TEAMS = 2;
constexpr int WBQ_BLOCK_BYTES = 128 * 256;
constexpr int WBQ_THREADS = (8 * WBQ_TEAMS + 1) * 32;
constexpr size_t WBQ_SMEM = size_t(WBQ_STAGES) * WBQ_BLOCK_BYTES + 2 * WBQ_STAGES * 8 + 128;

// Consumer side of the staged weight kernel.  Thread (warp w of its team, lane l) takes the
// 8-element segment l & 15 (16 B at byte 16 (l & 15)) of rows 16 w + 2 i + (l >> 4), i = 0..7:
// each LDS.128 of a warp reads two full 256-byte rows (every 8-lane phase 128 contiguous bytes:
// conflict-free, no lane permutation), and each 8-byte code store of a warp writes two full
// 128-byte code rows.  The tensor map zero-fills rows past n and columns past k, so the loads
// need no masks (zeros never raise the amax); the producer hands over (block row, block
// column, tensor) with the stage, so the consumers do no 64-bit division or tensor search.
template <bool kFanout>
__global__ void __launch_bounds__(WBQ_THREADS, 1) weight_blockwise_bulk_kernel(const __grid_constant__ WBatch bt,
                                                                               int32_t* __restrict__ nonfinite_flag) {
    extern __shared__ __align__(128) uint8_t wbq_smem[];
    __shared__ uint32_t red[WBQ_TEAMS][2][8];
    __shared__ uint2 wmeta[WBQ_STAGES];  // {block row, tensor << 24 | block column}
    __shared__ ScaleTables tabs;
    uint64_t* full = reinterpret_cast<uint64_t*>(wbq_smem + size_t(WBQ_STAGES) * WBQ_BLOCK_BYTES);
    uint64_t* empty = full + WBQ_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b0 = bt.nblocks * blockIdx.x / gridDim.x;
    const int64_t b1 = bt.nblocks * (blockIdx.x + 1) / gridDim.x;
    const int32_t nb = static_cast<int32_t>(b1 - b0);
    init_scale_tables(tabs);
    if (threadIdx.x == 0) {
        for (int s = 0; s < WBQ_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t ring = smem_u32(wbq_smem);
    if (warp == 8 * WBQ_TEAMS) {  // producer warp (one elected lane)
        if (lane != 0 || nb <= 0) return;
        int ti = 0;
        while (ti + 1 < bt.count && b0 >= bt.t[ti + 1].blk0) ++ti;
        const int64_t local = b0 - bt.t[ti].blk0;
        uint32_t bi = static_cast<uint32_t>(local / bt.t[ti].nbk);
        uint32_t bj = static_cast<uint32_t>(local - int64_t(bi) * bt.t[ti].nbk);
        uint32_t nbk = static_cast<uint32_t>(bt.t[ti].nbk);
        int64_t n = bt.t[ti].n;
        uint32_t s = 0, ph = 0;
        for (int32_t it = 0; it < nb; ++it) {
            mbar_wait(&empty[s], ph ^ 1u);
            wmeta[s] = make_uint2(bi, (static_cast<uint32_t>(ti) << 24) | bj);
            // the full box is counted even where it is zero-filled out of bounds
            mbar_arrive_expect_tx(&full[s], WBQ_BLOCK_BYTES);
            tma_load_2d_hint(wbq_smem + size_t(s) * WBQ_BLOCK_BYTES, &bt.tm[ti], &full[s],
                             static_cast<int32_t>(bj * 128), static_cast<int32_t>(bi * 128),
                             kL2EvictFirst);  // every byte is read once
            if (++bj == nbk) {
                bj = 0;
                if (int64_t(++bi) * 128 >= n && ti + 1 < bt.count) {
                    bi = 0;
                    ++ti;
                    nbk = static_cast<uint32_t>(bt.t[ti].nbk);
                    n = bt.t[ti].n;
                }
            }
            if (++s == WBQ_STAGES) {
                s = 0;
                ph ^= 1u;
            }
        }
        return;
    }
    const int team = warp >> 3, w = warp & 7;
    const uint32_t seg = static_cast<uint32_t>(lane & 15);
    const uint32_t r0 = static_cast<uint32_t>(w * 16 + (lane >> 4));  // first of this thread's rows
    int par = 0;
    uint32_t s = static_cast<uint32_t>(team), ph = 0;
    for (int32_t it = team; it < nb; it += WBQ_TEAMS) {
        mbar_wait(&full[s], ph);
        const uint2 md = wmeta[s];
        uint32_t v[8][4];
        const uint32_t src = ring + s * WBQ_BLOCK_BYTES + r0 * 256u + seg * 16u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3]) : "r"(src + i * 512u));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // the block is in registers: free the stage
        // block amax: max over sign-cleared BF16 bits (reading Q2), lanes, then the team's 8 warps
        uint32_t m2[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m2[i] = bmax_abs2(bmax_abs2(v[i][0], v[i][1]), bmax_abs2(v[i][2], v[i][3]));
        uint32_t a2 = bmax_abs2(bmax_abs2(bmax_abs2(m2[0], m2[1]), bmax_abs2(m2[2], m2[3])),
                                bmax_abs2(bmax_abs2(m2[4], m2[5]), bmax_abs2(m2[6], m2[7]))) &
                      0x7FFF7FFFu;
        uint32_t ab = __reduce_max_sync(0xFFFFFFFFu, max(a2 & 0xFFFFu, a2 >> 16));
        if (lane == 0) red[team][par][w] = ab;
        asm volatile("bar.sync %0, 256;" ::"r"(1 + team) : "memory");
        ab = red[team][par][0];
#pragma unroll
        for (int i = 1; i < 8; ++i) ab = max(ab, red[team][par][i]);
        const WTensor& t = bt.t[md.y >> 24];
        const uint32_t bi = md.x, bj = md.y & 0xFFFFFFu;
        const bool fast = ab >= kAmaxFastGuardBits && ab < kNonFiniteBits;  // block-uniform
        float sc, rc = 0.0f;
        if (fast)
            table_scale_rcp(tabs, ab, sc, rc);
        else
            sc = scale_from_amax_bits(ab);
        if (w == 0 && lane == 0) {
            float* sp = t.scales + int64_t(bi) * t.ld_s + bj;
            if (kFanout) {
                for (int dd = 0; dd < bt.ndest; ++dd)
                    *reinterpret_cast<float*>(reinterpret_cast<char*>(sp) + bt.ds[dd]) = sc;
            } else {
                *sp = sc;
            }
            if (ab >= kNonFiniteBits && nonfinite_flag != nullptr) *nonfinite_flag = 1;
        }
        const int64_t rows_left = t.n - int64_t(bi) * 128;
        const bool col_ok = int64_t(bj) * 128 + seg * 8 < t.k;
        uint8_t* qb = t.q + (int64_t(bi) * 128 + r0) * t.ld_q + int64_t(bj) * 128 + seg * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint2 c = fast ? encode8w<true>(v[i], sc, rc) : encode8w<false>(v[i], sc, 0.0f);
            if (col_ok && int64_t(r0) + 2 * i < rows_left) {
                uint8_t* dst = qb + int64_t(2 * i) * t.ld_q;
                if (kFanout) {
                    for (int dd = 0; dd < bt.ndest; ++dd) st_stream_v2(dst + bt.dq[dd], c.x, c.y);
                } else {
                    st_stream_v2(dst, c.x, c.y);
                }
            }
        }
        par ^= 1;
        s += WBQ_TEAMS;
        if (s >= WBQ_STAGES) {
            s -= WBQ_STAGES;
            ph ^= 1u;
        }
    }
}

int sm_count() {
    static int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return sms;
}

inline bool al(const void* p, uintptr_t a) { return reinterpret_cast<uintptr_t>(p) % a == 0; }

bool wide_ok(const WeightDesc& d) {
    return d.k % 16 == 0 && al(d.w, 32) && d.ld_w % 16 == 0 && al(d.q, 16) && d.ld_q % 16 == 0;
}

}  // namespace

cudaError_t launch_weight_blockwise_batch(const WeightDesc* descs, int count, int32_t* flag,
                                          cudaStream_t stream, int ndest, const int64_t* dq, const int64_t* ds) {
    // wide path for every aligned tensor, batched kMaxWeightBatch per launch
    WBatch bt{};
    bt.count = 0;
    bt.nblocks = 0;
    bt.ndest = ndest;
    for (int dd = 0; dd < ndest && dd < kMaxFanout; ++dd) {
        bt.dq[dd] = dq[dd];
        bt.ds[dd] = ds[dd];
    }
    if (ndest > 0)
        for (int i = 0; i < count; ++i)
            if (!wide_ok(descs[i])) return cudaErrorInvalidValue;  // fan-out runs on the wide path only
    // dev/test override: FP8Q_WEIGHT_KERNEL=wide | bulk forces that path (default: by size)
    static const int kernel_env = [] {
        const char* e = std::getenv("FP8Q_WEIGHT_KERNEL");
        return e == nullptr ? 0 : (e[0] == 'w' ? 1 : (e[0] == 'b' ? 2 : 0));
    }();
    const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encode_fn());
    // the bulk path wins on large batches (the per-layer sync launch: 11,776 blocks for a Qwen3-8B
    // layer) and loses a few % on a single small tensor (qkv: 1,536 blocks, ~10 per SM), where the
    // block-strided grid's register prefetch ramps up faster
    int64_t total_blocks = 0;
    for (int i = 0; i < count; ++i)
        if (wide_ok(descs[i])) total_blocks += ((descs[i].n + 127) / 128) * ((descs[i].k + 127) / 128);
    const bool bulk = encode != nullptr && kernel_env != 1 && (kernel_env == 2 || total_blocks >= 16LL * sm_count());
    auto flush = [&]() -> cudaError_t {
        if (bt.count == 0) return cudaSuccess;
        if (bulk) {
            static bool attr_done[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev >= 0 && dev < 64 && !attr_done[dev]) {
                cudaError_t ea = cudaFuncSetAttribute(weight_blockwise_bulk_kernel<false>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(WBQ_SMEM));
                if (ea == cudaSuccess)
                    ea = cudaFuncSetAttribute(weight_blockwise_bulk_kernel<true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(WBQ_SMEM));
                if (ea != cudaSuccess) return ea;
                attr_done[dev] = true;
            }
            const int64_t grid = bt.nblocks < sm_count() ? bt.nblocks : sm_count();
            if (bt.ndest > 0)
                weight_blockwise_bulk_kernel<true><<<static_cast<unsigned>(grid), WBQ_THREADS, WBQ_SMEM, stream>>>(
                    bt, flag);
            else
                weight_blockwise_bulk_kernel<false><<<static_cast<unsigned>(grid), WBQ_THREADS, WBQ_SMEM, stream>>>(
                    bt, flag);
            bt.count = 0;
            bt.nblocks = 0;
            return cudaGetLastError();
        }
        const int64_t cap = 2LL * sm_count();
        const int64_t grid = bt.nblocks < cap ? bt.nblocks : cap;
        if (grid > 0) {
            if (bt.ndest > 0)
                weight_blockwise_wide_kernel<true><<<static_cast<unsigned>(grid), 256, 0, stream>>>(bt, flag);
            else
                weight_blockwise_wide_kernel<false><<<static_cast<unsigned>(grid), 256, 0, stream>>>(bt, flag);
        }
        bt.count = 0;
        bt.nblocks = 0;
        return cudaGetLastError();
    };
    for (int i = 0; i < count; ++i) {
        const WeightDesc& d = descs[i];
        const int64_t nbn = (d.n + 127) / 128, nbk = (d.k + 127) / 128;
        const int64_t blocks = nbn * nbk;
        if (blocks == 0) continue;
        if (wide_ok(d)) {
            WTensor& t = bt.t[bt.count++];
            t.w = d.w;
            t.q = d.q;
            t.scales = d.scales;
            t.n = d.n;
            t.k = d.k;
            t.ld_w = d.ld_w;
            t.ld_q = d.ld_q;
            t.ld_s = d.ld_s;
            t.nbk = nbk;
            t.blk0 = bt.nblocks;
            if (bulk) {
                cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.k), static_cast<cuuint64_t>(d.n)};
                cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.ld_w) * 2};
                cuuint32_t box[2] = {128, 128};
                cuuint32_t estr[2] = {1, 1};
                const CUresult r = encode(&bt.tm[bt.count - 1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                          const_cast<uint16_t*>(d.w), dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
            }
            bt.nblocks += blocks;
            if (bt.count == kMaxWeightBatch) {
                cudaError_t e = flush();
                if (e != cudaSuccess) return e;
            }
        } else {
            if (blocks > 0x7FFFFFFFLL) return cudaErrorInvalidConfiguration;
            weight_blockwise_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
                d.w, d.n, d.k, d.ld_w, d.q, d.ld_q, d.scales, d.ld_s, nbk, flag);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    return flush();
}

int weight_batch_launches(const WeightDesc* descs, int count) {
    int wide = 0, narrow = 0;
    for (int i = 0; i < count; ++i) {
        const WeightDesc& d = descs[i];
        if (d.n == 0 || d.k == 0) continue;
        if (wide_ok(d)) ++wide; else ++narrow;
    }
    return narrow + (wide + kMaxWeightBatch - 1) / kMaxWeightBatch;
}

namespace {
// a3 on raw fp32 pairs: the quantizers' cvt_e4m3x2 helper (element i -> byte i), grid-stride.
__global__ void __launch_bounds__(256) e4m3_encode_kernel(const float2* __restrict__ x, int64_t pairs,
                                                          uint16_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < pairs;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = x[i];
        out[i] = static_cast<uint16_t>(cvt_e4m3x2(v.x, v.y));
    }
}
}  // namespace

cudaError_t launch_e4m3_encode(const float* x, int64_t n, uint8_t* codes, cudaStream_t stream) {
    const int64_t pairs = n / 2;
    int64_t blocks = (pairs + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    e4m3_encode_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        reinterpret_cast<const float2*>(x), pairs, reinterpret_cast<uint16_t*>(codes));
    return cudaGetLastError();
}

cudaError_t launch_weight_blockwise(const uint16_t* w, int64_t n, int64_t k, int64_t ld_w,
                                    uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                    int32_t* flag, cudaStream_t stream) {
    const WeightDesc d{w, n, k, ld_w, q, ld_q, scales, ld_s};
    return launch_weight_blockwise_batch(&d, 1, flag, stream);
}

namespace {
// The staged kernel's requirements: x 16-byte aligned with ld_x % 8 == 0 (TMA / bulk copies),
// codes 16-byte aligned with ld_q % 16 == 0 (16-byte stores), items < 2^31 per tensor.
bool act_staged_ok(const ActDesc& d) {
    const int64_t groups = d.k / 128;
    return al(d.x, 16) && d.ld_x % 8 == 0 && al(d.q, 16) && d.ld_q % 16 == 0 &&
           d.m * ((groups + 15) / 16) < (1LL << 31);
}
int act_kernel_env() {  // dev: FP8Q_ACT_KERNEL=wide selects the warp-persistent path
    static const int v = [] {
        const char* e = std::getenv("FP8Q_ACT_KERNEL");
        return (e != nullptr && e[0] == 'w') ? 1 : 0;
    }();
    return v;
}

cudaError_t launch_act_unstaged(const ActDesc& d, int32_t* flag, cudaStream_t stream) {
    const int64_t groups = d.k / 128;
    if (al(d.x, 32) && d.ld_x % 16 == 0 && al(d.q, 16) && d.ld_q % 16 == 0) {
        const int64_t wchunks = (groups + 15) / 16;
        const int64_t witems = d.m * wchunks;
        const int64_t wblocks = (witems + 7) / 8;
        const int64_t grid = wblocks < 2LL * sm_count() ? wblocks : 2LL * sm_count();
        const cudaError_t e = launch_pdl(act_per_token_group_wide_kernel, static_cast<unsigned>(grid), 256, 0, stream,
                                         d.x, d.ld_x, d.q, d.ld_q, d.scales, d.ld_s, groups, wchunks, witems, flag);
        if (e != cudaSuccess) return e;
    } else {
        const int64_t chunks = (groups + 7) / 8;
        const int64_t blocks = (d.m * chunks + 7) / 8;
        if (blocks > 0x7FFFFFFFLL) return cudaErrorInvalidConfiguration;
        act_per_token_group_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
            d.x, d.m, d.k, d.ld_x, d.q, d.ld_q, d.scales, d.ld_s, chunks, flag);
    }
    return cudaGetLastError();
}
}  // namespace

int act_batch_launches(const ActDesc* descs, int count) {
    int staged = 0, other = 0;
    for (int i = 0; i < count; ++i) {
        if (descs[i].m == 0 || descs[i].k == 0) continue;
        if (act_kernel_env() == 0 && act_staged_ok(descs[i]) && descs[i].m > 256) ++staged; else ++other;
    }
    return other + (staged + kMaxActBatch - 1) / kMaxActBatch;
}

cudaError_t launch_act_batch(const ActDesc* descs, int count, int32_t* flag, cudaStream_t stream) {
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !attr_done[dev]) {
        cudaError_t ea = cudaFuncSetAttribute(act_per_token_group_bulk_kernel<false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ABQ_SMEM));
        if (ea == cudaSuccess)
            ea = cudaFuncSetAttribute(act_per_token_group_bulk_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ABQ_SMEM));
        if (ea != cudaSuccess) return ea;
        attr_done[dev] = true;
    }
    // dev A/B: FP8Q_ACT_LOAD=bulk keeps the cp.async.bulk copies
    static const bool act_tma_env = [] {
        const char* e = std::getenv("FP8Q_ACT_LOAD");
        return !(e != nullptr && e[0] == 'b');
    }();
    const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encode_fn());
    const bool use_tma = act_tma_env && encode != nullptr;
    ABatch ab{};
    ab.count = 0;
    ab.units = 0;
    auto flush = [&]() -> cudaError_t {
        if (ab.count == 0 || ab.units == 0) {
            ab.count = 0;
            ab.units = 0;
            return cudaSuccess;
        }
        const int64_t per_cta_min = 2;  // small inputs: fewer CTAs, each a few stages
        int64_t grid = (ab.units + per_cta_min - 1) / per_cta_min;
        grid = grid < sm_count() ? grid : sm_count();
        const cudaError_t e =
            use_tma ? launch_pdl(act_per_token_group_bulk_kernel<true>, static_cast<unsigned>(grid), ABQ_THREADS,
                                 ABQ_SMEM, stream, ab, flag)
                    : launch_pdl(act_per_token_group_bulk_kernel<false>, static_cast<unsigned>(grid), ABQ_THREADS,
                                 ABQ_SMEM, stream, ab, flag);
        if (e != cudaSuccess) return e;
        ab.count = 0;
        ab.units = 0;
        return cudaGetLastError();
    };
    for (int i = 0; i < count; ++i) {
        const ActDesc& d = descs[i];
        if (d.m == 0 || d.k == 0) continue;
        // decode-sized inputs (<= 256 tokens) take the register path: no shared memory, so under
        // PDL its CTAs fit beside the previous GEMM's and the quantization starts the moment
        // that GEMM retires
        if (act_kernel_env() != 0 || !act_staged_ok(d) || d.m <= 256) {
            cudaError_t e = launch_act_unstaged(d, flag, stream);
            if (e != cudaSuccess) return e;
            continue;
        }
        const int64_t groups = d.k / 128;
        ATensor& t = ab.t[ab.count];
        t.x = d.x;
        t.q = d.q;
        t.scales = d.scales;
        t.ld_x = d.ld_x;
        t.ld_q = d.ld_q;
        t.ld_s = d.ld_s;
        t.groups = groups;
        t.m = d.m;
        t.chunks = static_cast<int32_t>((groups + 15) / 16);
        t.unit0 = ab.units;
        if (use_tma) {
            cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(groups), static_cast<cuuint64_t>(d.m)};
            cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(d.ld_x) * 2};
            cuuint32_t box[3] = {128, 16, static_cast<cuuint32_t>(ABQ_ITEMS)};
            cuuint32_t estr[3] = {1, 1, 1};
            if (encode(&ab.tm[ab.count], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(d.x), dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return cudaErrorInvalidValue;
        }
        ab.units += ((d.m + ABQ_ITEMS - 1) / ABQ_ITEMS) * t.chunks;
        if (++ab.count == kMaxActBatch) {
            cudaError_t e = flush();
            if (e != cudaSuccess) return e;
        }
    }
    return flush();
}

cudaError_t launch_act_per_token_group(const uint16_t* x, int64_t m, int64_t k, int64_t ld_x,
                                       uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                       int32_t* flag, cudaStream_t stream) {
    const ActDesc d{x, m, k, ld_x, q, ld_q, scales, ld_s};
    return launch_act_batch(&d, 1, flag, stream);
}

}  // namespace fp8q

FP8Q_TRACE_DUMP_FN(fp8q_trace_dump_quant)

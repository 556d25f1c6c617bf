// mx.cu -- SURVEY §8(f) NEXT-4: the MXFP8 variant (readings X1-X3).
//
//   mx_quantize     E4M3 codes with E8M0 power-of-two scales on 1x32 blocks along K:
//                   s = 2^e, e = the smallest integer (>= -127) with 448 * 2^e >= amax (no
//                   element saturates), amax == 0 -> e = 0; code = E4M3_RNE(x / s) -- the
//                   division by a power of two is exact, so the quantizer needs no division.
//   fp8_mx_gemm     D = sum_k dec(a) 2^ea dec(b) 2^eb with tcgen05.mma.kind::mxf8f6f4
//                   .block_scale: the tensor core applies the scales per 32-K sub-block, the
//                   accumulator stays in TMEM for the whole K loop (no per-k-block promotion
//                   round trip through registers -- the TMEM-read traffic that bounds the
//                   fp32-scale kernel of gemm.cu).
//
// Scale-factor layout ("native", chosen so a k-block's factors are one contiguous 512-byte
// chunk per 128 rows): byte (r, j) -- row r, 32-K sub-block j -- lives at
//     ((r / 128) * (K / 128) + j / 4) * 512 + (r % 128) * 4 + j % 4.
// TMEM layout the block-scaled MMA (cta_group::1, M = 128) reads, established with
// tools/mx_probe.py on the B200: SFA of row m at lane m of column m / 32 (byte = the MMA's
// a_sf_id) -- the kernel writes row m's word into all four columns of lane m, which also
// covers that reading; SFB of row n at column n / 32, lane n % 32 of EVERY 32-lane quarter
// (each quarter of the datapath reads its own copy; byte = b_sf_id); SF columns must be even.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <mutex>

#include "ptx.cuh"
#include "quant_kernels.h"

namespace fp8q {
namespace {

// ------------------------------------------------------------------------- quantizer
constexpr uint32_t kMxNonFinite = 0x7F80u;

// e for a block amax given as sign-cleared BF16 bits (X2)
__device__ __forceinline__ int mx_exp(uint32_t a) {
    if (a == 0u) return 0;
    const int E = static_cast<int>(a >> 7);
    if (E == 0) return -127;  // subnormal amax < 2^-126: 448 * 2^-127 already covers it
    // amax = 1.m * 2^(E-127); 448 = 1.75 * 2^8: e = E - 135, plus 1 if the significand > 1.75
    const int e = E - 135 + ((a & 0x7Fu) > 0x60u ? 1 : 0);
    return e < -127 ? -127 : e;
}

// one warp per (row, 256-column chunk); lane l holds columns 8l..8l+7 of the chunk, four lanes
// per 32-block
__global__ void __launch_bounds__(256) mx_quantize_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t k,
                                                          int64_t ld_x, uint8_t* __restrict__ q, int64_t ld_q,
                                                          uint8_t* __restrict__ sf, int32_t* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t chunks = k / 256 + (k % 256 ? 1 : 0);
    const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (item >= rows * chunks) return;
    const int64_t row = item / chunks;
    const int64_t col = (item - row * chunks) * 256 + lane * 8;
    const bool live = col < k;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (live) v = *reinterpret_cast<const uint4*>(x + row * ld_x + col);
    const uint32_t m = 0x7FFF7FFFu;
    uint32_t a = __vmaxu2(__vmaxu2(v.x & m, v.y & m), __vmaxu2(v.z & m, v.w & m));
    a = max(a & 0xFFFFu, a >> 16);
    a = max(a, __shfl_xor_sync(0xFFFFFFFFu, a, 1));
    a = max(a, __shfl_xor_sync(0xFFFFFFFFu, a, 2));
    if (!live) return;
    const int e = mx_exp(a);
    const float inv = __uint_as_float(static_cast<uint32_t>(127 - e) << 23);  // 2^-e, exact
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t wa = w[2 * i], wb = w[2 * i + 1];
        const uint32_t lo = cvt_e4m3x2(__uint_as_float(wa << 16) * inv, __uint_as_float(wa & 0xFFFF0000u) * inv);
        const uint32_t hi = cvt_e4m3x2(__uint_as_float(wb << 16) * inv, __uint_as_float(wb & 0xFFFF0000u) * inv);
        c[i] = lo | (hi << 16);
    }
    st_stream_v2(q + row * ld_q + col, c[0], c[1]);
    if ((lane & 3) == 0) {
        const int64_t j = col / 32;
        sf[((row / 128) * (k / 128) + j / 4) * 512 + (row % 128) * 4 + (j % 4)] = static_cast<uint8_t>(e + 127);
        if (a >= kMxNonFinite && flag != nullptr) *flag = 1;
    }
}

// ------------------------------------------------------------------------- GEMM
constexpr int MX_BM = 128;
constexpr int MX_BN = 256;
constexpr int MX_BK = 128;
constexpr int MX_STAGES = 4;
constexpr int MX_A_TILE = MX_BM * MX_BK;               // 16 KB
constexpr int MX_B_TILE = MX_BN * MX_BK;               // 32 KB
constexpr int MX_SFA_BYTES = 512;                      // 128 rows x 4 sub-blocks
constexpr int MX_SFB_BYTES = 1024;                     // 256 rows x 4 sub-blocks
constexpr int MX_STAGE = MX_A_TILE + MX_B_TILE + MX_SFA_BYTES + MX_SFB_BYTES;
constexpr int MX_THREADS = 320;  // warps 0-3 SF writers, 4-7 epilogue, 8 TMA, 9 MMA
constexpr int MX_SF_SLOTS = 8;   // TMEM scale-factor ring (k-blocks)
constexpr int MX_SF_COL0 = 256;  // TMEM: accumulator columns [0, 256), SF slots from 256
constexpr int MX_RASTER = 16;    // m-tiles per raster band
constexpr size_t MX_SMEM = 1024 + size_t(MX_STAGES) * MX_STAGE + 256;

// block-scaled idesc: E4M3 x E4M3, K-major, N >> 3 at [17,23), E8M0 scales (bit 23),
// M >> 4 at [24,29), b_sf_id at [4,6), a_sf_id at [29,31)
__host__ __device__ constexpr uint32_t mx_idesc(uint32_t sf_id) {
    return (sf_id << 4) | ((MX_BN >> 3) << 17) | (1u << 23) | ((MX_BM >> 4) << 24) | (sf_id << 29);
}

struct MxParams {
    const uint8_t* sfa;  // native layout
    const uint8_t* sfb;
    void* d;
    int64_t ld_d;
    int out_f32;
    int m, n, num_kb, tiles_m, tiles_n;
};

__device__ __forceinline__ bool mx_tile(const MxParams& p, int t, int& mt, int& nt) {
    const int per_band = MX_RASTER * p.tiles_n;
    const int band = t / per_band;
    const int r = t - band * per_band;
    const int rows_in = min(MX_RASTER, p.tiles_m - band * MX_RASTER);
    if (rows_in <= 0) return false;
    mt = band * MX_RASTER + r % rows_in;
    nt = r / rows_in;
    return true;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_st_x4(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v), "r"(v), "r"(v),
                 "r"(v)
                 : "memory");
}
__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                       uint32_t tsfa, uint32_t tsfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(tsfa), "r"(tsfb)
        : "memory");
}

__global__ void __launch_bounds__(MX_THREADS, 1)
    fp8_mx_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const MxParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smA = smem;
    uint8_t* smB = smA + MX_STAGES * MX_A_TILE;
    uint8_t* smSA = smB + MX_STAGES * MX_B_TILE;
    uint8_t* smSB = smSA + MX_STAGES * MX_SFA_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smSB + MX_STAGES * MX_SFB_BYTES);
    uint64_t* empty = full + MX_STAGES;        // MMA consumed A/B (commit)
    uint64_t* sempty = empty + MX_STAGES;      // SF writers consumed the stage's factors
    uint64_t* sf_full = sempty + MX_STAGES;    // [slots] factors are in TMEM
    uint64_t* sf_empty = sf_full + MX_SF_SLOTS;  // [slots] the MMA reading them completed
    uint64_t* tfull = sf_empty + MX_SF_SLOTS;  // accumulator complete
    uint64_t* tempty = tfull + 1;              // accumulator drained by the epilogue
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = p.tiles_m * p.tiles_n;
    if (threadIdx.x == 0) {
        for (int s = 0; s < MX_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&sempty[s], 4);
        }
        for (int s = 0; s < MX_SF_SLOTS; ++s) {
            mbar_init(&sf_full[s], 4);
            mbar_init(&sf_empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 4);
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

    if (warp == 8) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            uint32_t it = 0;
            int mt, nt;
            for (int t = blockIdx.x; t < tiles && mx_tile(p, t, mt, nt); t += gridDim.x) {
                for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                    const uint32_t s = it % MX_STAGES, ph = (it / MX_STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_wait(&sempty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[s], MX_STAGE);
                    tma_load_2d(smA + s * MX_A_TILE, &tmA, &full[s], kb * MX_BK, mt * MX_BM);
                    tma_load_2d(smB + s * MX_B_TILE, &tmB, &full[s], kb * MX_BK, nt * MX_BN);
                    bulk_g2s(smSA + s * MX_SFA_BYTES, p.sfa + (int64_t(mt) * p.num_kb + kb) * 512, 512, &full[s]);
                    const int64_t nb0 = int64_t(nt) * 2;
                    bulk_g2s(smSB + s * MX_SFB_BYTES, p.sfb + (nb0 * p.num_kb + kb) * 512, 512, &full[s]);
                    bulk_g2s(smSB + s * MX_SFB_BYTES + 512, p.sfb + ((nb0 + 1) * p.num_kb + kb) * 512, 512, &full[s]);
                }
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            uint32_t it = 0, tile_no = 0;
            int mt, nt;
            for (int t = blockIdx.x; t < tiles && mx_tile(p, t, mt, nt); t += gridDim.x, ++tile_no) {
                mbar_wait(tempty, (tile_no & 1u) ^ 1u);  // the epilogue drained the accumulator
                tc_fence_after();
                for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                    const uint32_t s = it % MX_STAGES, ph = (it / MX_STAGES) & 1u;
                    const uint32_t f = it % MX_SF_SLOTS, fph = (it / MX_SF_SLOTS) & 1u;
                    mbar_wait(&full[s], ph);
                    mbar_wait(&sf_full[f], fph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smA + s * MX_A_TILE), b0 = smem_u32(smB + s * MX_B_TILE);
                    const uint32_t tsfa = tmem + MX_SF_COL0 + f * 16, tsfb = tsfa + 8;
#pragma unroll
                    for (int kk = 0; kk < MX_BK / 32; ++kk)
                        mma_mx(tmem, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32), mx_idesc(kk),
                               (kb > 0 || kk > 0) ? 1u : 0u, tsfa, tsfb);
                    mma_commit(&empty[s]);
                    mma_commit(&sf_empty[f]);
                }
                mma_commit(tfull);
            }
        }
    } else if (warp < 4) {
        // ---------------------------------------------------------------- SF writers
        // warp q writes its 32-lane quarter: SFA of rows 32q + lane (one column), and the
        // full SFB (8 columns: n = 32c + lane), which every quarter needs its own copy of.
        const int q = warp;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        uint32_t it = 0;
        int mt, nt;
        for (int t = blockIdx.x; t < tiles && mx_tile(p, t, mt, nt); t += gridDim.x) {
            for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                const uint32_t s = it % MX_STAGES, ph = (it / MX_STAGES) & 1u;
                const uint32_t f = it % MX_SF_SLOTS, fph = (it / MX_SF_SLOTS) & 1u;
                mbar_wait(&full[s], ph);
                const uint32_t wa = reinterpret_cast<const uint32_t*>(smSA + s * MX_SFA_BYTES)[q * 32 + lane];
                uint32_t wb[8];
                const uint32_t* sb = reinterpret_cast<const uint32_t*>(smSB + s * MX_SFB_BYTES);
#pragma unroll
                for (int c = 0; c < 8; ++c) wb[c] = sb[c * 32 + lane];
                __syncwarp();
                if (lane == 0) mbar_arrive(&sempty[s]);  // the stage's factors are in registers
                mbar_wait(&sf_empty[f], fph ^ 1u);      // the MMA that read this slot completed
                tc_fence_after();
                const uint32_t col = tmem + lane_base + MX_SF_COL0 + f * 16;
                tmem_st_x4(col, wa);  // row m's word in columns 0-3 of lane m (see header)
                tmem_st_x8(col + 8, wb);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sf_full[f]);
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue (warps 4-7)
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        uint32_t tile_no = 0;
        int mt, nt;
        for (int t = blockIdx.x; t < tiles && mx_tile(p, t, mt, nt); t += gridDim.x, ++tile_no) {
            mbar_wait(tfull, tile_no & 1u);
            tc_fence_after();
            const int64_t row = int64_t(mt) * MX_BM + q * 32 + lane;
            const bool row_ok = row < p.m;
#pragma unroll 1
            for (int c = 0; c < MX_BN / 32; ++c) {
                float v[32];
                tmem_ld_32x32b_x32(tmem + lane_base + c * 32, v);
                tmem_wait_ld();
                if (c == MX_BN / 32 - 1) {  // the whole accumulator is in registers / stored
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty);
                }
                const int64_t col0 = int64_t(nt) * MX_BN + c * 32;
                if (!row_ok || col0 >= p.n) continue;
                if (p.out_f32) {
                    float* d = static_cast<float*>(p.d) + row * p.ld_d + col0;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        if (col0 + j < p.n)
                            st_v4(d + j, __float_as_uint(v[j]), __float_as_uint(v[j + 1]), __float_as_uint(v[j + 2]),
                                  __float_as_uint(v[j + 3]));
                } else {
                    __nv_bfloat16* d = static_cast<__nv_bfloat16*>(p.d) + row * p.ld_d + col0;
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        if (col0 + j >= p.n) break;
                        uint32_t o[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            __nv_bfloat162 h = __floats2bfloat162_rn(v[j + 2 * i], v[j + 2 * i + 1]);
                            o[i] = *reinterpret_cast<uint32_t*>(&h);
                        }
                        st_v4(d + j, o[0], o[1], o[2], o[3]);
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int mx_sms() {
    static int v = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    return v;
}

}  // namespace

size_t mx_sf_bytes(int64_t rows, int64_t k) { return static_cast<size_t>((rows + 127) / 128) * (k / 128) * 512; }

cudaError_t launch_mx_quantize(const uint16_t* x, int64_t rows, int64_t k, int64_t ld_x, uint8_t* q, int64_t ld_q,
                               uint8_t* sf, int32_t* flag, cudaStream_t stream) {
    if (rows == 0 || k == 0) return cudaSuccess;
    const int64_t items = rows * ((k + 255) / 256);
    const int64_t blocks = (items + 7) / 8;
    if (blocks > 0x7FFFFFFFLL) return cudaErrorInvalidConfiguration;
    mx_quantize_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(x, rows, k, ld_x, q, ld_q, sf, flag);
    return cudaGetLastError();
}

cudaError_t launch_fp8_mx_gemm(const uint8_t* a, int64_t ld_a, const uint8_t* sfa, const uint8_t* b, int64_t ld_b,
                               const uint8_t* sfb, void* d, int64_t ld_d, bool out_f32, int64_t m, int64_t n,
                               int64_t k, void* encode_fn, cudaStream_t stream) {
    if (m == 0 || n == 0) return cudaSuccess;
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
    if (encode == nullptr) return cudaErrorNotSupported;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(fp8_mx_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(MX_SMEM));
    });
    if (attr != cudaSuccess) return attr;
    CUtensorMap tmA, tmB;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_a)};
        cuuint32_t box[2] = {MX_BK, MX_BM};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_b)};
        cuuint32_t box[2] = {MX_BK, MX_BN};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(b), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    MxParams p;
    p.sfa = sfa;
    p.sfb = sfb;
    p.d = d;
    p.ld_d = ld_d;
    p.out_f32 = out_f32 ? 1 : 0;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.num_kb = static_cast<int>(k / MX_BK);
    p.tiles_m = static_cast<int>((m + MX_BM - 1) / MX_BM);
    p.tiles_n = static_cast<int>((n + MX_BN - 1) / MX_BN);
    const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n;
    const unsigned grid = static_cast<unsigned>(tiles < mx_sms() ? tiles : mx_sms());
    fp8_mx_gemm_kernel<<<grid, MX_THREADS, MX_SMEM, stream>>>(tmA, tmB, p);
    return cudaGetLastError();
}

}  // namespace fp8q

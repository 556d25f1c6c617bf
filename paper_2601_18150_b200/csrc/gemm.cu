// gemm.cu -- blockwise-scaled FP8 GEMM for sm_100a (tcgen05 + TMA + TMEM), dense and grouped.
//
// Computes ("W8A8 ... DeepGEMM"; granularity PAPER.md:233)
//     D[m,n] = sum_kb  (sa[kb][m] * sb[n/128][kb]) * P_kb[m,n],
//     P_kb[m,n] = sum_{k in kb} dec(a[m,k]) * dec(b[n,k])      (128-deep k-block kb)
// The scales are arbitrary fp32 (amax/448), so they cannot ride in the tensor core's UE8M0
// block-scale path: every k-block's partial P_kb is produced by the tensor core in TMEM and
// promoted by CUDA-core FMAs into an fp32 register accumulator ("scale promotion").
//
// CTA = 12 warps (3 warpgroups), persistent over 128x256 output tiles (M-fastest order so
// concurrent CTAs share B tiles and the whole A panel stays L2-resident).  Warpgroup 0 gives
// registers away (setmaxnreg.dec 56) and warpgroups 1-2 take them (setmaxnreg.inc 224): the
// register file is per SM sub-partition, so 3 warps x 168 at launch become 56 + 224 + 224.
//   warp 0        TMA producer: per k-block, A 128x128 B and B 256x128 B into a 4-stage ring
//                 (128-byte swizzle), mbarrier full/empty handshake with the MMA warp.
//   warp 1        TMEM owner (512 columns) and MMA issuer: 4 x tcgen05.mma.kind::f8f6f4
//                 (M=128, N=256, K=32) per k-block into TMEM buffer (it % 2), fresh
//                 accumulation per k-block; tcgen05.commit frees the smem stage and
//                 publishes the partial.
//   warps 2,3     idle (they only donate registers).
//   warps 4..11   promotion/epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (its 32 rows),
//                 warps 4-7 columns 0-127 and 8-11 columns 128-255 (one weight n-block each,
//                 so one scale product per thread per k-block).  acc += P_kb * (sa*sb) with
//                 packed FFMA2; the TMEM buffer is released as soon as it is read, so the
//                 tensor core fills the other buffer while the FMAs run.  After the last
//                 k-block each thread writes its row segment (BF16 = RNE of the F32 value).
// Determinism: fixed k-block order, no atomics.  DESIGN.md §5.2 has the roofline analysis.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <mutex>

#include "ptx.cuh"
#include "quant_kernels.h"

namespace fp8q {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;
constexpr int STAGES = 4;
constexpr int A_TILE = BM * BK;  // bytes (E4M3)
constexpr int B_TILE = BN * BK;
constexpr int STAGE_BYTES = A_TILE + B_TILE;
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int TMEM_COLS = 512;  // 2 partial buffers x 256 fp32 columns
constexpr int NUM_EPI_WARPS = 8;
constexpr int RASTER_GM = 16;  // m-tiles per raster band
constexpr uint32_t IDESC = idesc_e4m3_f32(BM, BN);
constexpr size_t SMEM_BYTES = 1024 + size_t(STAGES) * STAGE_BYTES + 256;

struct KParams {
    const float* sa;
    int64_t ld_sa;
    const float* sb;
    int64_t ld_sb;
    int64_t stride_sb;
    void* d;
    int64_t ld_d;
    int out_f32;
    int64_t m;
    int64_t n;
    int num_kb;
    int num_n_tiles;
    const int32_t* offsets;  // nullptr: one group of m rows
    int groups;
};

// Walks the (group, m-tile, n-tile) sequence; t must increase between calls.
struct TileCursor {
    int g;
    int64_t base;   // first linear tile index of group g
    int64_t row0;   // first A/D row of group g
    int64_t rows;   // rows in group g
    int64_t mtiles; // ceil(rows / BM)
    __device__ void load(const KParams& p) {
        if (p.offsets != nullptr) {
            row0 = p.offsets[g];
            rows = static_cast<int64_t>(p.offsets[g + 1]) - row0;
        } else {
            row0 = 0;
            rows = p.m;
        }
        mtiles = (rows + BM - 1) / BM;
    }
    __device__ void init(const KParams& p) {
        g = 0;
        base = 0;
        if (p.groups > 0) load(p);
    }
    // Returns false when t is past the last tile.
    __device__ bool seek(const KParams& p, int64_t t, int& mt, int& nt) {
        if (g >= p.groups) return false;
        while (t >= base + mtiles * p.num_n_tiles) {
            base += mtiles * p.num_n_tiles;
            if (++g >= p.groups) return false;
            load(p);
        }
        // Grouped raster: bands of RASTER_GM m-tiles; inside a band m is fastest, so the ~148
        // concurrent tiles cover a compact RASTER_GM x ~9 block of the output and both the A
        // band and the B tiles they touch stay L2-resident (K = 12288 would otherwise re-read A).
        const int64_t l = t - base;
        const int64_t band = l / (int64_t(RASTER_GM) * p.num_n_tiles);
        const int64_t r = l - band * (int64_t(RASTER_GM) * p.num_n_tiles);
        const int64_t gm = min(int64_t(RASTER_GM), mtiles - band * RASTER_GM);
        mt = static_cast<int>(band * RASTER_GM + r % gm);
        nt = static_cast<int>(r / gm);
        return true;
    }
};

__device__ __forceinline__ void ffma2(float2& acc, const float2 v, const float f) {
    uint64_t a = *reinterpret_cast<uint64_t*>(&acc);
    const uint64_t x = *reinterpret_cast<const uint64_t*>(&v);
    const float2 ff = make_float2(f, f);
    const uint64_t s = *reinterpret_cast<const uint64_t*>(&ff);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(x), "l"(s));
    acc = *reinterpret_cast<float2*>(&a);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    fp8_block_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB, const KParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smA = smem;
    uint8_t* smB = smem + STAGES * A_TILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], NUM_EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < EPI_WARP0) regs_dec<56>();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            TileCursor cur;
            cur.init(p);
            uint32_t it = 0;
            int mt, nt;
            for (int64_t t = blockIdx.x; cur.seek(p, t, mt, nt); t += gridDim.x) {
                const int32_t arow = static_cast<int32_t>(cur.row0 + int64_t(mt) * BM);
                const int32_t brow = nt * BN;
                for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&empty[stage], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                    tma_load_2d(smA + stage * A_TILE, &tmA, &full[stage], kb * BK, arow);
                    tma_load_3d(smB + stage * B_TILE, &tmB, &full[stage], kb * BK, brow, cur.g);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
            TileCursor cur;
            cur.init(p);
            uint32_t it = 0;
            int mt, nt;
            for (int64_t t = blockIdx.x; cur.seek(p, t, mt, nt); t += gridDim.x) {
                for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    const uint32_t buf = it & 1u;
                    const uint32_t bph = (it >> 1) & 1u;
                    mbar_wait(&tempty[buf], bph ^ 1u);  // promotion warps drained this buffer
                    mbar_wait(&full[stage], ph);        // TMA landed A and B
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smA + stage * A_TILE);
                    const uint32_t b0 = smem_u32(smB + stage * B_TILE);
                    const uint32_t d = tmem + buf * BN;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk)
                        mma_f8f6f4(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32),
                                   IDESC, kk > 0 ? 1u : 0u);
                    mma_commit(&empty[stage]);
                    mma_commit(&tfull[buf]);
                }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------------------------------------------------------- promotion warps
        regs_inc<224>();
        const int h = (warp - EPI_WARP0) >> 2;  // column half: n-block 2*nt + h
        const int qd = warp & 3;         // TMEM lane quarter this warp may access
        const int r_in_tile = qd * 32 + lane;
        const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
        float2 acc[64];
        TileCursor cur;
        cur.init(p);
        uint32_t it = 0;
        int mt, nt;
        for (int64_t t = blockIdx.x; cur.seek(p, t, mt, nt); t += gridDim.x) {
            const int64_t rloc = int64_t(mt) * BM + r_in_tile;
            const bool row_ok = rloc < cur.rows;
            const int64_t row = cur.row0 + rloc;
            const int64_t nb = int64_t(nt) * 2 + h;
            const bool nb_ok = nb * 128 < p.n;
            const bool live = row_ok && nb_ok;
            const float* sap = p.sa + row;
            const float* sbp = p.sb + int64_t(cur.g) * p.stride_sb + nb * p.ld_sb;
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = make_float2(0.f, 0.f);
            // Scale prefetch two k-blocks ahead; the raw values are only multiplied when used,
            // so the load latency never sits between the TMEM-full wait and the FMAs.
            float sa0 = 0.f, sb0 = 0.f, sa1 = 0.f, sb1 = 0.f;
            if (live) {
                sa0 = __ldg(sap);
                sb0 = __ldg(sbp);
                if (p.num_kb > 1) {
                    sa1 = __ldg(sap + p.ld_sa);
                    sb1 = __ldg(sbp + 1);
                }
            }
            for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                const float f = sa0 * sb0;
                sa0 = sa1;
                sb0 = sb1;
                if (live && kb + 2 < p.num_kb) {
                    sa1 = __ldg(sap + int64_t(kb + 2) * p.ld_sa);
                    sb1 = __ldg(sbp + kb + 2);
                }
                const uint32_t buf = it & 1u;
                const uint32_t bph = (it >> 1) & 1u;
                mbar_wait(&tfull[buf], bph);
                tc_fence_after();
                const uint32_t taddr = tmem + (static_cast<uint32_t>(qd * 32) << 16) + buf * BN + h * 128;
#pragma unroll
                for (int c = 0; c < 4; c += 2) {
                    float v0[32], v1[32];
                    tmem_ld_32x32b_x32(taddr + c * 32, v0);
                    tmem_ld_32x32b_x32(taddr + (c + 1) * 32, v1);
                    tmem_wait_ld();
                    if (c == 2) {  // whole partial read: hand the buffer back to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        ffma2(acc[c * 16 + j], make_float2(v0[2 * j], v0[2 * j + 1]), f);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        ffma2(acc[(c + 1) * 16 + j], make_float2(v1[2 * j], v1[2 * j + 1]), f);
                }
            }
            if (live) {
                const int64_t col0 = nb * 128;
                if (p.out_f32) {
                    float* drow = static_cast<float*>(p.d) + row * p.ld_d + col0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (col0 + j * 4 < p.n)
                            st_v4(drow + j * 4, __float_as_uint(acc[2 * j].x), __float_as_uint(acc[2 * j].y),
                                  __float_as_uint(acc[2 * j + 1].x), __float_as_uint(acc[2 * j + 1].y));
                    }
                } else {
                    __nv_bfloat16* drow = static_cast<__nv_bfloat16*>(p.d) + row * p.ld_d + col0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (col0 + j * 8 < p.n) {
                            uint32_t w[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[4 * j + e].x, acc[4 * j + e].y);
                                w[e] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                            st_v4(drow + j * 8, w[0], w[1], w[2], w[3]);
                        }
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(*reinterpret_cast<volatile uint32_t*>(tmem_slot), TMEM_COLS);
    }
}

// ------------------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

struct DeviceInfo {
    int sms = 0;
    bool attr_set = false;
};
DeviceInfo g_dev[64];
std::mutex g_dev_mu;

cudaError_t device_info(int& sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo& di = g_dev[dev];
    if (!di.attr_set) {
        e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fp8_block_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SMEM_BYTES));
        if (e != cudaSuccess) return e;
        di.attr_set = true;
    }
    sms = di.sms;
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_fp8_block_gemm(const GemmArgs& a, cudaStream_t stream, int* launches) {
    *launches = 0;
    if (a.m == 0 || a.n == 0 || a.groups == 0) return cudaSuccess;
    auto encode = tensor_map_encoder();
    if (encode == nullptr) return cudaErrorNotSupported;
    int sms = 0;
    cudaError_t e = device_info(sms);
    if (e != cudaSuccess) return e;

    CUtensorMap tmA, tmB;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_a)};
        cuuint32_t box[2] = {BK, BM};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.a), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {
        const int64_t g = a.offsets != nullptr ? a.groups : 1;
        const int64_t sb = (g > 1) ? a.stride_b : a.ld_b * a.n;
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.n),
                              static_cast<cuuint64_t>(g)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.ld_b), static_cast<cuuint64_t>(sb)};
        cuuint32_t box[3] = {BK, BN, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(a.b), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }

    KParams p;
    p.sa = a.sa;
    p.ld_sa = a.ld_sa;
    p.sb = a.sb;
    p.ld_sb = a.ld_sb;
    p.stride_sb = a.stride_sb;
    p.d = a.d;
    p.ld_d = a.ld_d;
    p.out_f32 = a.out_f32 ? 1 : 0;
    p.m = a.m;
    p.n = a.n;
    p.num_kb = static_cast<int>(a.k / BK);
    p.num_n_tiles = static_cast<int>((a.n + BN - 1) / BN);
    p.offsets = a.offsets;
    p.groups = a.offsets != nullptr ? a.groups : 1;

    int64_t grid = sms;
    if (a.offsets == nullptr) {
        const int64_t tiles = ((a.m + BM - 1) / BM) * p.num_n_tiles;
        grid = tiles < sms ? tiles : sms;
    }
    fp8_block_gemm_kernel<<<static_cast<unsigned>(grid), NUM_THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
    *launches = 1;
    return cudaGetLastError();
}

}  // namespace fp8q

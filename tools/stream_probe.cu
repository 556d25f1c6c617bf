// stream_probe.cu -- dev microbenchmark: how fast can a persistent grid stream an FP8 weight
// matrix [N, K] into shared memory, by access pattern (no compute: the consumer frees each
// stage the moment it lands).  Each CTA streams an equal contiguous range of (128-row tile,
// 128-byte k-block) units, k fastest, as the decode GEMM's stream-K does.
//   mode 0: one 2-D TMA box (128 rows x 128 B) per unit from the row-major [N, K] matrix
//           (the decode GEMM's weight loads today)
//   mode 1: one contiguous 16 KB cp.async.bulk per unit (a block-tiled layout: every 128 x 128
//           block stored contiguously)
//   mode 2: one 2-D TMA box of 128 rows x 256 B (two k-blocks) per two units
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

using namespace fp8q;

namespace {
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* w,
                                                        int mode, int stages, int64_t tiles, int64_t kbs) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int unit_bytes = mode == 2 ? 32768 : 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(stages) * unit_bytes);
    uint64_t* empty = full + stages;
    const int64_t per = mode == 2 ? 2 : 1;
    const int64_t total = tiles * kbs / per;
    const int64_t u0 = total * blockIdx.x / gridDim.x, u1 = total * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0, ph = 0;
        for (int64_t u = u0; u < u1; ++u) {
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], unit_bytes);
            const int64_t tile = (u * per) / kbs, kb = (u * per) - tile * kbs;
            if (mode == 1)
                bulk_g2s(smem_u32(sm + size_t(s) * unit_bytes), w + u * 16384, 16384, &full[s]);
            else
                tma_load_2d(sm + size_t(s) * unit_bytes, &tm, &full[s], static_cast<int32_t>(kb * 128),
                            static_cast<int32_t>(tile * 128));
            if (++s == static_cast<uint32_t>(stages)) {
                s = 0;
                ph ^= 1u;
            }
        }
    } else if (threadIdx.x == 32) {
        uint32_t s = 0, ph = 0;
        for (int64_t u = u0; u < u1; ++u) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == static_cast<uint32_t>(stages)) {
                s = 0;
                ph ^= 1u;
            }
        }
    }
}
}  // namespace

extern "C" int stream_probe(int mode, int stages, const void* w, long long n, long long k, int grid, void* stream) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return 1;
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(k)};
    cuuint32_t box[2] = {mode == 2 ? 256u : 128u, 128u};
    cuuint32_t estr[2] = {1, 1};
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(w), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, mode == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 2;
    const int unit_bytes = mode == 2 ? 32768 : 16384;
    const size_t smem = size_t(stages) * unit_bytes + 2 * stages * 8 + 64;
    if (cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 3;
    stream_kernel<<<grid, 64, smem, static_cast<cudaStream_t>(stream)>>>(tm, static_cast<const uint8_t*>(w), mode,
                                                                          stages, n / 128, k / 128);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

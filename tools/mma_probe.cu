// mma_probe.cu -- dev microbenchmark: the per-k-block cost of the prefill GEMM's MMA issue
// sequence with operands resident in shared memory (no TMA, no promotion, no buffer waits).
// One cluster = one CTA pair (or grid/2 pairs); the leader's thread issues NKB k-blocks of
// 4 x tcgen05.mma (K = 32 each) into TMEM buffer kb % 2 and records clock64 before the first
// MMA and after the final commit has landed.
//   mode 0: cta_group::2, M=256 N=256, 2 multicast commits per k-block (the kernel's sequence)
//   mode 1: same MMAs, one commit at the very end
//   mode 2: same MMAs, one multicast commit per k-block
//   mode 3: cta_group::2, M=256 N=128 (kind 1128), 2 commits per k-block
//   mode 4: mode 0, but the 4 MMAs of a k-block read 4 different 32-byte K slices of a
//           stage ring of 4 stages (descriptor address moves like the real kernel)
//   mode 5: cta_group::1 (no pair), M=128 N=256, 2 commits per k-block (each CTA issues)
//   modes 6 / 7 / 8: as mode 5 with N = 16 / 64 / 128 (the decode kernel's swap-AB shapes)
//   mode 9: mode 6 plus the decode issuer's per-k-block bookkeeping: two mbarrier waits on
//           (already completed) barriers and a tcgen05 fence before the MMAs
#include <cstdint>

#include "ptx.cuh"

using namespace fp8q;

namespace {
__device__ __forceinline__ void mma_f8f6f4_1(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit_1(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_probe_kernel(int mode, int nkb, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smA = smem;                  // 4 stages x 16 KB
    uint8_t* smB = smem + 4 * 16384;      // 4 stages x 16 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 8 * 16384);  // [0..7] per-kb, [8] final
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 16);
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < 8 * 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x38383838u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
        mbar_init(&bars[12], 1);
        mbar_init(&bars[13], 1);
        mbar_arrive(&bars[12]);
        mbar_arrive(&bars[13]);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    const bool pair = mode < 5;
    if (warp == 1) {
        if (pair)
            tmem_alloc_pair(slot, 512);
        else
            tmem_alloc(slot, 512);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(slot);
    const bool issuer = threadIdx.x == 0 && (rank == 0 || !pair);
    if (issuer) {
        const uint32_t N = mode == 3 ? 128 : (mode == 6 || mode == 9) ? 16 : mode == 7 ? 64 : mode == 8 ? 128 : 256;
        const uint32_t idesc = pair ? idesc_e4m3_f32(256, N) : idesc_e4m3_f32(128, N);
        const long long t0 = clock64();
        for (int kb = 0; kb < nkb; ++kb) {
            const uint32_t st = mode == 4 ? static_cast<uint32_t>(kb & 3) : 0u;
            const uint32_t a0 = smem_u32(smA + st * 16384), b0 = smem_u32(smB + st * 16384);
            const uint32_t d = tmem + static_cast<uint32_t>(kb & 1) * N;
            if (mode == 9) {
                mbar_wait(&bars[12], 0);  // completed at init: the waits return at once
                mbar_wait(&bars[13], 0);
                tc_fence_after();
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (pair)
                    mma_f8f6f4_pair(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32), idesc,
                                    kk > 0 ? 1u : 0u);
                else
                    mma_f8f6f4_1(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32), idesc,
                                 kk > 0 ? 1u : 0u);
            }
            if (mode == 0 || mode == 3 || mode == 4) {
                mma_commit_pair(&bars[kb & 3], 0x3);
                mma_commit_pair(&bars[4 + (kb & 1)], 0x3);
            } else if (mode == 2) {
                mma_commit_pair(&bars[kb & 3], 0x3);
            } else if (mode >= 5) {
                commit_1(&bars[kb & 3]);
                commit_1(&bars[4 + (kb & 1)]);
            }
        }
        if (pair)
            mma_commit_pair(&bars[8], 0x3);
        else
            commit_1(&bars[8]);
        mbar_wait(&bars[8], 0);
        const long long t1 = clock64();
        out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    }
    if (pair && rank == 1 && threadIdx.x == 0) mbar_wait(&bars[8], 0);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        if (pair)
            tmem_dealloc_pair(tmem, 512);
        else
            tmem_dealloc(tmem, 512);
    }
}

extern "C" int mma_probe(int mode, int nkb, int grid, unsigned long long* out_dev) {
    const int smem = 8 * 16384 + 1024 + 256;
    cudaFuncSetAttribute(mma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_probe_kernel<<<grid, 128, smem>>>(mode, nkb, out_dev);
    return static_cast<int>(cudaDeviceSynchronize());
}

// mx_probe.cu -- dev experiment (not part of the product): where does
// tcgen05.mma.kind::mxf8f6f4.block_scale read its UE8M0 scale factors from TMEM?
// A and B are all-ones E4M3 (0x38), so D[m][n] = sum over the K=32 chunk of
// 2^(sfa(m)-127) * 2^(sfb(n)-127) = 32 * 2^(sfa(m) + sfb(n) - 254): the scale each output
// used is readable from D.  Scale words are written to TMEM with tcgen05.st from registers
// (lane l of the CTA writes sfa_words[l] at column SFA_COL, sfb_words[l] at SFB_COL).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC
//        -I paper_2601_18150_b200/csrc tools/mx_probe.cu -o tools/libmxprobe.so
#include <cstdint>

#include "ptx.cuh"

using namespace fp8q;

namespace {
constexpr int SFA_COL = 256;
constexpr int SFB_COL = 320;

__device__ __forceinline__ void tmem_st_x1(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void probe_kernel(const uint32_t* sfa_words, const uint32_t* sfb_words, int n_dim, uint32_t idesc,
                             uint32_t sfa_col_off, uint32_t sfb_col_off, float* d_out) {
    __shared__ __align__(1024) uint8_t smB[256 * 128];  // all 0x38: A reads its first 128 rows
    uint8_t* smA = smB;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * 128; i += blockDim.x) smB[i] = 0x38;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    // scale words: warp w owns TMEM lanes 32w..32w+31
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    for (int c = 0; c < 8; ++c) {
        tmem_st_x1(tmem + lane_base + SFA_COL + c, sfa_words[c * 128 + threadIdx.x]);
        tmem_st_x1(tmem + lane_base + SFB_COL + c, sfb_words[c * 128 + threadIdx.x]);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint64_t da = smem_desc_k_sw128(smem_u32(smA));
        const uint64_t db = smem_desc_k_sw128(smem_u32(smB));
        const uint32_t tsfa = tmem + SFA_COL + sfa_col_off;
        const uint32_t tsfb = tmem + SFB_COL + sfb_col_off;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(0u), "r"(tsfa), "r"(tsfb)
            : "memory");
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c = 0; c < n_dim; c += 32) {
        float v[32];
        tmem_ld_32x32b_x32(tmem + lane_base + c, v);
        tmem_wait_ld();
        for (int j = 0; j < 32; ++j) d_out[(warp * 32 + lane) * 256 + c + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}
}  // namespace

extern "C" int mx_probe(const uint32_t* sfa_words, const uint32_t* sfb_words, int n_dim, uint32_t idesc,
                        uint32_t sfa_col_off, uint32_t sfb_col_off, float* d_out) {
    probe_kernel<<<1, 128>>>(sfa_words, sfb_words, n_dim, idesc, sfa_col_off, sfb_col_off, d_out);
    return static_cast<int>(cudaDeviceSynchronize());
}

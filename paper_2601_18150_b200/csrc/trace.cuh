// Dev-only launch timeline (compiled in only with -DFP8Q_TRACE, i.e. the separate
// libfp8q_trace.so that `build.py --trace` writes; the production library has none of it).
// Each event is one 16-byte record {tag, cta | smid << 20, event, globaltimer} appended to a
// per-translation-unit ring; `fp8q_trace_dump_<tu>` copies it out and resets it.
#pragma once
#include <cstdint>

#ifdef FP8Q_TRACE
#define FP8Q_TRACE_CAP (1u << 20)
namespace fp8q_trace {
static __device__ uint32_t g_n;
static __device__ uint4 g_rec[FP8Q_TRACE_CAP];
__device__ __forceinline__ void rec(uint32_t tag, uint32_t ev) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint32_t i = atomicAdd(&g_n, 1u);
    if (i < FP8Q_TRACE_CAP)
        g_rec[i] = make_uint4(tag, blockIdx.x | (smid << 20), ev | (static_cast<uint32_t>(t >> 32) << 8),
                              static_cast<uint32_t>(t));
}
inline int dump(void* host, uint32_t cap, uint32_t* n) {
    uint32_t cnt = 0;
    if (cudaMemcpyFromSymbol(&cnt, g_n, 4) != cudaSuccess) return -1;
    if (cnt > FP8Q_TRACE_CAP) cnt = FP8Q_TRACE_CAP;
    if (cnt > cap) cnt = cap;
    if (cnt && cudaMemcpyFromSymbol(host, g_rec, size_t(cnt) * 16) != cudaSuccess) return -1;
    *n = cnt;
    const uint32_t z = 0;
    return cudaMemcpyToSymbol(g_n, &z, 4) == cudaSuccess ? 0 : -1;
}
}  // namespace fp8q_trace
#define FP8Q_TREC(tag, ev) fp8q_trace::rec((tag), (ev))
#define FP8Q_TRACE_DUMP_FN(name) \
    extern "C" int name(void* host, uint32_t cap, uint32_t* n) { return fp8q_trace::dump(host, cap, n); }
#else
#define FP8Q_TREC(tag, ev) ((void)0)
#define FP8Q_TRACE_DUMP_FN(name)
#endif

// pdl.cuh -- programmatic dependent launch (PDL) for the element-map kernels that sit between
// two GEMMs on the rollout forward (activation quantizers, producer-fused quantizers): they
// trigger the dependent launch at entry, so the next kernel (the decode GEMM prefetches its
// weights before its own griddepcontrol.wait) starts while they run, and they wait for the
// preceding grid -- complete, its memory visible -- before touching their inputs or outputs.
// Launched without the attribute, both instructions are no-ops.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace fp8q {

__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Launch with the programmatic-stream-serialization attribute.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace fp8q

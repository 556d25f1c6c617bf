// quant_kernels.h -- internal launch entry points (C++), wrapped by the C-ABI in capi.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fp8q {

constexpr int kMaxWeightBatch = 16;  // tensors per batched weight-quantization launch
constexpr int kMaxFanout = 8;        // destinations of the fan-out (NEXT-1) weight quantizer

struct WeightDesc {
    const uint16_t* w;
    int64_t n, k, ld_w;
    uint8_t* q;
    int64_t ld_q;
    float* scales;
    int64_t ld_s;
};

// All descs in as few launches as possible (kMaxWeightBatch wide-path tensors per launch;
// tensors that miss the wide path's alignment get their own launch of the general kernel).
cudaError_t launch_weight_blockwise_batch(const WeightDesc* descs, int count, int32_t* flag,
                                          cudaStream_t stream, int ndest = 0, const int64_t* dq = nullptr,
                                          const int64_t* ds = nullptr);
int weight_batch_launches(const WeightDesc* descs, int count);

cudaError_t launch_weight_blockwise(const uint16_t* w, int64_t n, int64_t k, int64_t ld_w,
                                    uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                    int32_t* flag, cudaStream_t stream);

// a3 element encode on raw fp32 pairs (e4m3_encode_f32): the quantizers' cvt helper.
cudaError_t launch_e4m3_encode(const float* x, int64_t n, uint8_t* codes, cudaStream_t stream);

cudaError_t launch_act_per_token_group(const uint16_t* x, int64_t m, int64_t k, int64_t ld_x,
                                       uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                       int32_t* flag, cudaStream_t stream);

// Several activation tensors in as few launches as possible (kMaxActBatch staged-path tensors
// per persistent launch; tensors that miss the staged path's alignment get their own launch).
constexpr int kMaxActBatch = 8;
struct ActDesc {
    const uint16_t* x;
    int64_t m, k, ld_x;
    uint8_t* q;
    int64_t ld_q;
    float* scales;
    int64_t ld_s;
};
cudaError_t launch_act_batch(const ActDesc* descs, int count, int32_t* flag, cudaStream_t stream);
int act_batch_launches(const ActDesc* descs, int count);

struct GemmArgs {
    const uint8_t* a;
    int64_t ld_a;
    const float* sa;
    int64_t ld_sa;
    const uint8_t* b;
    int64_t ld_b;
    int64_t stride_b;  // bytes between groups' B matrices (grouped); ignored if groups == 1
    const float* sb;
    int64_t ld_sb;
    int64_t stride_sb;  // elements between groups' scale grids
    void* d;
    int64_t ld_d;
    bool out_f32;
    int64_t m, n, k;
    const int32_t* offsets;  // device [groups + 1] or nullptr (dense)
    int32_t groups;
    void* workspace;         // split-K workspace (zero-filled before first use), may be null
    size_t workspace_bytes;
    // fp8_linear_dynamic at m <= 16 (decode): BF16 activations quantized inside the GEMM (a, sa unused)
    const uint16_t* x_bf16 = nullptr;
    int64_t ld_x = 0;
    int32_t* nonfinite_flag = nullptr;
};
// whether the decode kernel can quantize this linear's activations itself (m <= 16, the CTA's
// k-blocks' codes fit its shared memory); the caller then sets x_bf16 / ld_x
bool skinny_fused_act_applies(const GemmArgs& a);

// Decode-sized dense GEMMs (1 <= m <= kSkinnyMaxM) run the swap-AB kernel of gemm_skinny.cu
// (m > 128 only where its cluster split-K mode applies).
constexpr int kSkinnyMaxM = 256;
bool skinny_gemm_applies(const GemmArgs& a);
// The CTA-pair kernel would split its tail-wave tiles along K for this dense shape (gemm.cu
// plan_split); at decode M = 256 that wins over the swap-AB kernel, which then steps aside.
bool pair_tail_split_applies(int64_t m, int64_t n, int64_t k, size_t workspace_bytes);
size_t skinny_workspace_bytes(int64_t m, int64_t n, int64_t k);
cudaError_t launch_fp8_gemm_skinny(const GemmArgs& a, void* encode_fn, cudaStream_t stream);

// Bytes of workspace with which launch_fp8_block_gemm uses split-K for this shape (0: never).
size_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, bool grouped);

// Enqueue the tcgen05 blockwise-scaled FP8 GEMM.  Returns cudaSuccess or the first error.
cudaError_t launch_fp8_block_gemm(const GemmArgs& args, cudaStream_t stream, int* launches);

// NEXT-2 producer-fused quantizers (producers.cu).
cudaError_t launch_rmsnorm_quantize(const uint16_t* x, const uint16_t* gamma, float eps, int64_t m, int64_t k,
                                    int64_t ld_x, uint8_t* q, int64_t ld_q, float* scales, int64_t ld_s,
                                    uint16_t* y, int64_t ld_y, int32_t* flag, cudaStream_t stream);
cudaError_t launch_silu_mul_quantize(const uint16_t* gu, int64_t m, int64_t inter, int64_t ld_gu, uint8_t* q,
                                     int64_t ld_q, float* scales, int64_t ld_s, uint16_t* y, int64_t ld_y,
                                     int32_t* flag, cudaStream_t stream);

// NEXT-3 FP8 KV cache (kv.cu).
cudaError_t launch_kv_amax(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, uint32_t* amax_bits,
                           int32_t* flag, cudaStream_t stream);
cudaError_t launch_kv_scale(const uint32_t* amax_bits, int64_t n, float* scales, cudaStream_t stream);
cudaError_t launch_kv_append(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x, const float* scale,
                             const int32_t* slots, uint8_t* cache, int64_t ld_c, int64_t num_slots,
                             uint32_t* saturated, int32_t* flag, cudaStream_t stream);

// NEXT-4 MXFP8 variant (mx.cu).
size_t mx_sf_bytes(int64_t rows, int64_t k);
cudaError_t launch_mx_quantize(const uint16_t* x, int64_t rows, int64_t k, int64_t ld_x, uint8_t* q, int64_t ld_q,
                               uint8_t* sf, int32_t* flag, cudaStream_t stream);
cudaError_t launch_fp8_mx_gemm(const uint8_t* a, int64_t ld_a, const uint8_t* sfa, const uint8_t* b, int64_t ld_b,
                               const uint8_t* sfb, void* d, int64_t ld_d, bool out_f32, int64_t m, int64_t n,
                               int64_t k, void* encode_fn, cudaStream_t stream);
void* tensor_map_encode_fn();


}  // namespace fp8q

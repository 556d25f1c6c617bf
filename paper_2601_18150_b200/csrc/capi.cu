// capi.cu -- the extern "C" boundary declared in include/fp8q.h: argument validation,
// status codes, dispatch to the sm_100a kernels.  No allocation, no host sync, no exceptions.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/fp8q.h"
#include "quant_kernels.h"

namespace {

std::atomic<int64_t> g_launches{0};

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

fp8q_status check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return FP8Q_ECUDA;
    static std::atomic<int> cached[64];  // 0 unknown, 1 ok, 2 unsupported
    if (dev < 0 || dev >= 64) return FP8Q_EUNSUPPORTED;
    int c = cached[dev].load();
    if (c == 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
            return FP8Q_ECUDA;
        c = (major == 10 && minor == 0) ? 1 : 2;  // built for sm_100a only
        cached[dev].store(c);
    }
    return c == 1 ? FP8Q_OK : FP8Q_EUNSUPPORTED;
}

thread_local cudaError_t g_last_cuda = cudaSuccess;
fp8q_status from_cuda(cudaError_t e) {
    if (e != cudaSuccess) g_last_cuda = e;
    return e == cudaSuccess ? FP8Q_OK : FP8Q_ECUDA;
}

}  // namespace

extern "C" {

const char* fp8q_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda); }

const char* fp8q_status_string(fp8q_status s) {
    switch (s) {
        case FP8Q_OK: return "FP8Q_OK";
        case FP8Q_EINVAL: return "FP8Q_EINVAL: null pointer, negative dimension or leading dimension too small";
        case FP8Q_ESHAPE: return "FP8Q_ESHAPE: shape constraint violated (k % 128, k % 8, n % 8, groups)";
        case FP8Q_EALIGN: return "FP8Q_EALIGN: pointer or leading-dimension alignment requirement violated";
        case FP8Q_ECUDA: return "FP8Q_ECUDA: a CUDA runtime call failed";
        case FP8Q_EUNSUPPORTED: return "FP8Q_EUNSUPPORTED: device is not sm_100 (B200)";
        case FP8Q_EWORKSPACE: return "FP8Q_EWORKSPACE: workspace too small";
    }
    return "FP8Q_UNKNOWN_STATUS";
}

int32_t fp8q_version(void) { return 10000; }

int64_t fp8q_kernel_launches(void) { return g_launches.load(); }

fp8q_status e4m3_encode_f32(const float* x, int64_t n, uint8_t* codes, void* stream) {
    if (n < 0) return FP8Q_EINVAL;
    if (n == 0) return FP8Q_OK;
    if (x == nullptr || codes == nullptr) return FP8Q_EINVAL;
    if (n % 2 != 0) return FP8Q_ESHAPE;
    if (!aligned(x, 8) || !aligned(codes, 2)) return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_e4m3_encode(x, n, codes, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}


static fp8q_status check_weight(const void* w_bf16, int64_t n, int64_t k, int64_t ld_w, const uint8_t* codes,
                                int64_t ld_q, const float* scales, int64_t ld_s) {
    if (n < 0 || k < 0) return FP8Q_EINVAL;
    if (ld_w < k || ld_q < k || ld_s < (k + 127) / 128) return FP8Q_EINVAL;
    if (n == 0 || k == 0) return FP8Q_OK;
    if (w_bf16 == nullptr || codes == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (k % 8 != 0) return FP8Q_ESHAPE;
    if (!aligned(w_bf16, 16) || ld_w % 8 != 0 || !aligned(codes, 8) || ld_q % 8 != 0 || !aligned(scales, 4))
        return FP8Q_EALIGN;
    return FP8Q_OK;
}

fp8q_status quantize_weight_blockwise(const void* w_bf16, int64_t n, int64_t k, int64_t ld_w,
                                      uint8_t* codes, int64_t ld_q, float* scales, int64_t ld_s,
                                      int32_t* nonfinite_flag, void* stream) {
    fp8q_status st = check_weight(w_bf16, n, k, ld_w, codes, ld_q, scales, ld_s);
    if (st != FP8Q_OK || n == 0 || k == 0) return st;
    if (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)) return FP8Q_EALIGN;
    st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_weight_blockwise(static_cast<const uint16_t*>(w_bf16), n, k, ld_w,
                                                  codes, ld_q, scales, ld_s, nonfinite_flag,
                                                  static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status quantize_weight_blockwise_batched(const fp8q_weight_tensor* tensors, int32_t count,
                                              int32_t* nonfinite_flag, void* stream) {
    if (count < 0 || (count > 0 && tensors == nullptr)) return FP8Q_EINVAL;
    if (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)) return FP8Q_EALIGN;
    for (int32_t i = 0; i < count; ++i) {
        const fp8q_weight_tensor& t = tensors[i];
        fp8q_status st = check_weight(t.w_bf16, t.n, t.k, t.ld_w, t.codes, t.ld_q, t.scales, t.ld_s);
        if (st != FP8Q_OK) return st;
    }
    if (count == 0) return FP8Q_OK;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    // chunks of kMaxWeightBatch descriptors on the stack (no host allocation, nothing can throw)
    fp8q::WeightDesc d[fp8q::kMaxWeightBatch];
    for (int32_t base = 0; base < count; base += fp8q::kMaxWeightBatch) {
        const int32_t c = count - base < fp8q::kMaxWeightBatch ? count - base : fp8q::kMaxWeightBatch;
        for (int32_t i = 0; i < c; ++i) {
            const fp8q_weight_tensor& t = tensors[base + i];
            d[i] = fp8q::WeightDesc{static_cast<const uint16_t*>(t.w_bf16), t.n, t.k, t.ld_w, t.codes, t.ld_q,
                                    t.scales, t.ld_s};
        }
        cudaError_t e = fp8q::launch_weight_blockwise_batch(d, c, nonfinite_flag, static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return from_cuda(e);
        g_launches.fetch_add(fp8q::weight_batch_launches(d, c));
    }
    return FP8Q_OK;
}

fp8q_status quantize_weight_blockwise_fanout(const fp8q_weight_tensor* tensors, int32_t count, int32_t num_dest,
                                             const int64_t* codes_delta, const int64_t* scales_delta,
                                             int32_t* nonfinite_flag, void* stream) {
    if (count < 0 || (count > 0 && tensors == nullptr)) return FP8Q_EINVAL;
    if (num_dest < 1 || num_dest > fp8q::kMaxFanout || codes_delta == nullptr || scales_delta == nullptr)
        return FP8Q_EINVAL;
    if (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)) return FP8Q_EALIGN;
    for (int32_t d = 0; d < num_dest; ++d)
        if (codes_delta[d] % 16 != 0 || scales_delta[d] % 4 != 0) return FP8Q_EALIGN;
    for (int32_t i = 0; i < count; ++i) {
        const fp8q_weight_tensor& t = tensors[i];
        fp8q_status st = check_weight(t.w_bf16, t.n, t.k, t.ld_w, t.codes, t.ld_q, t.scales, t.ld_s);
        if (st != FP8Q_OK) return st;
        // the fan-out runs on the wide path only: k % 16, 32-byte-aligned w, ld_w % 16,
        // 16-byte-aligned codes, ld_q % 16
        if (t.k % 16 != 0 || !aligned(t.w_bf16, 32) || t.ld_w % 16 != 0 || !aligned(t.codes, 16) || t.ld_q % 16 != 0)
            return FP8Q_EUNSUPPORTED;
    }
    if (count == 0) return FP8Q_OK;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    fp8q::WeightDesc d[fp8q::kMaxWeightBatch];
    for (int32_t base = 0; base < count; base += fp8q::kMaxWeightBatch) {
        const int32_t c = count - base < fp8q::kMaxWeightBatch ? count - base : fp8q::kMaxWeightBatch;
        for (int32_t i = 0; i < c; ++i) {
            const fp8q_weight_tensor& t = tensors[base + i];
            d[i] = fp8q::WeightDesc{static_cast<const uint16_t*>(t.w_bf16), t.n, t.k, t.ld_w, t.codes, t.ld_q,
                                    t.scales, t.ld_s};
        }
        cudaError_t e = fp8q::launch_weight_blockwise_batch(d, c, nonfinite_flag, static_cast<cudaStream_t>(stream),
                                                            num_dest, codes_delta, scales_delta);
        if (e != cudaSuccess) return from_cuda(e);
        g_launches.fetch_add(fp8q::weight_batch_launches(d, c));
    }
    return FP8Q_OK;
}

fp8q_status quantize_act_per_token_group(const void* x_bf16, int64_t m, int64_t k, int64_t ld_x,
                                         uint8_t* codes, int64_t ld_q, float* scales, int64_t ld_s,
                                         int32_t* nonfinite_flag, void* stream) {
    if (m < 0 || k < 0) return FP8Q_EINVAL;
    if (ld_x < k || ld_q < k || ld_s < m) return FP8Q_EINVAL;
    if (k % 128 != 0) return FP8Q_ESHAPE;
    if (m == 0 || k == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || codes == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 16) || ld_x % 8 != 0 || !aligned(codes, 8) || ld_q % 8 != 0 ||
        !aligned(scales, 4) || ld_s % 4 != 0 ||
        (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)))
        return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_act_per_token_group(static_cast<const uint16_t*>(x_bf16), m, k, ld_x,
                                                     codes, ld_q, scales, ld_s, nonfinite_flag,
                                                     static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

static fp8q_status check_act(const void* x_bf16, int64_t m, int64_t k, int64_t ld_x, const uint8_t* codes,
                             int64_t ld_q, const float* scales, int64_t ld_s) {
    if (m < 0 || k < 0) return FP8Q_EINVAL;
    if (ld_x < k || ld_q < k || ld_s < m) return FP8Q_EINVAL;
    if (k % 128 != 0) return FP8Q_ESHAPE;
    if (m == 0 || k == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || codes == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 16) || ld_x % 8 != 0 || !aligned(codes, 8) || ld_q % 8 != 0 || !aligned(scales, 4) ||
        ld_s % 4 != 0)
        return FP8Q_EALIGN;
    return FP8Q_OK;
}

fp8q_status quantize_act_per_token_group_batched(const fp8q_act_tensor* tensors, int32_t count,
                                                 int32_t* nonfinite_flag, void* stream) {
    if (count < 0 || (count > 0 && tensors == nullptr)) return FP8Q_EINVAL;
    if (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)) return FP8Q_EALIGN;
    for (int32_t i = 0; i < count; ++i) {
        const fp8q_act_tensor& t = tensors[i];
        fp8q_status st = check_act(t.x_bf16, t.m, t.k, t.ld_x, t.codes, t.ld_q, t.scales, t.ld_s);
        if (st != FP8Q_OK) return st;
    }
    if (count == 0) return FP8Q_OK;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    fp8q::ActDesc d[fp8q::kMaxActBatch];
    for (int32_t base = 0; base < count; base += fp8q::kMaxActBatch) {
        const int32_t c = count - base < fp8q::kMaxActBatch ? count - base : fp8q::kMaxActBatch;
        for (int32_t i = 0; i < c; ++i) {
            const fp8q_act_tensor& t = tensors[base + i];
            d[i] = fp8q::ActDesc{static_cast<const uint16_t*>(t.x_bf16), t.m, t.k, t.ld_x, t.codes, t.ld_q,
                                 t.scales, t.ld_s};
        }
        cudaError_t e = fp8q::launch_act_batch(d, c, nonfinite_flag, static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return from_cuda(e);
        g_launches.fetch_add(fp8q::act_batch_launches(d, c));
    }
    return FP8Q_OK;
}

static fp8q_status check_act_out(int64_t m, int64_t k, const uint8_t* codes, int64_t ld_q, const float* scales,
                                 int64_t ld_s, const void* y, int64_t ld_y, const int32_t* flag) {
    if (ld_q < k || ld_s < m || (y != nullptr && ld_y < k)) return FP8Q_EINVAL;
    if (codes == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (!aligned(codes, 8) || ld_q % 8 != 0 || !aligned(scales, 4) || ld_s % 4 != 0 ||
        (y != nullptr && (!aligned(y, 16) || ld_y % 8 != 0)) || (flag != nullptr && !aligned(flag, 4)))
        return FP8Q_EALIGN;
    return FP8Q_OK;
}

fp8q_status rmsnorm_quantize_act_per_token_group(const void* x_bf16, const void* gamma_bf16, float eps,
                                                 int64_t m, int64_t k, int64_t ld_x, uint8_t* codes,
                                                 int64_t ld_q, float* scales, int64_t ld_s, void* y_bf16,
                                                 int64_t ld_y, int32_t* nonfinite_flag, void* stream) {
    if (m < 0 || k < 0 || ld_x < k) return FP8Q_EINVAL;
    if (k % 128 != 0 || k > 4096) return FP8Q_ESHAPE;
    if (m == 0 || k == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || gamma_bf16 == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 16) || !aligned(gamma_bf16, 16) || ld_x % 8 != 0) return FP8Q_EALIGN;
    fp8q_status st = check_act_out(m, k, codes, ld_q, scales, ld_s, y_bf16, ld_y, nonfinite_flag);
    if (st != FP8Q_OK) return st;
    st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_rmsnorm_quantize(static_cast<const uint16_t*>(x_bf16),
                                                  static_cast<const uint16_t*>(gamma_bf16), eps, m, k, ld_x, codes,
                                                  ld_q, scales, ld_s, static_cast<uint16_t*>(y_bf16), ld_y,
                                                  nonfinite_flag, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status silu_mul_quantize_act_per_token_group(const void* gate_up_bf16, int64_t m, int64_t inter,
                                                  int64_t ld_gu, uint8_t* codes, int64_t ld_q, float* scales,
                                                  int64_t ld_s, void* y_bf16, int64_t ld_y,
                                                  int32_t* nonfinite_flag, void* stream) {
    if (m < 0 || inter < 0 || ld_gu < 2 * inter) return FP8Q_EINVAL;
    if (inter % 128 != 0) return FP8Q_ESHAPE;
    if (m == 0 || inter == 0) return FP8Q_OK;
    if (gate_up_bf16 == nullptr) return FP8Q_EINVAL;
    if (!aligned(gate_up_bf16, 16) || ld_gu % 8 != 0) return FP8Q_EALIGN;
    fp8q_status st = check_act_out(m, inter, codes, ld_q, scales, ld_s, y_bf16, ld_y, nonfinite_flag);
    if (st != FP8Q_OK) return st;
    st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_silu_mul_quantize(static_cast<const uint16_t*>(gate_up_bf16), m, inter, ld_gu,
                                                   codes, ld_q, scales, ld_s, static_cast<uint16_t*>(y_bf16), ld_y,
                                                   nonfinite_flag, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status kv_amax_update(const void* x_bf16, int64_t rows, int64_t cols, int64_t ld_x, uint32_t* amax_bits,
                           int32_t* flag, void* stream) {
    if (rows < 0 || cols < 0 || ld_x < cols) return FP8Q_EINVAL;
    if (rows == 0 || cols == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || amax_bits == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 2) || !aligned(amax_bits, 4) || !aligned(flag, 4)) return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_kv_amax(static_cast<const uint16_t*>(x_bf16), rows, cols, ld_x, amax_bits, flag,
                                         static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status kv_scale_from_amax(const uint32_t* amax_bits, int64_t count, float* scales, void* stream) {
    if (count < 0) return FP8Q_EINVAL;
    if (count == 0) return FP8Q_OK;
    if (amax_bits == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (!aligned(amax_bits, 4) || !aligned(scales, 4)) return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_kv_scale(amax_bits, count, scales, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status kv_quantize_append(const void* x_bf16, int64_t rows, int64_t cols, int64_t ld_x, const float* scale,
                               const int32_t* slots, uint8_t* cache, int64_t ld_cache, int64_t num_slots,
                               uint32_t* saturated, int32_t* flag, void* stream) {
    if (rows < 0 || cols < 0 || ld_x < cols || ld_cache < cols || num_slots < 0) return FP8Q_EINVAL;
    if (slots == nullptr && rows > num_slots) return FP8Q_ESHAPE;
    if (rows == 0 || cols == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || scale == nullptr || cache == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 2) || !aligned(scale, 4) || !aligned(slots, 4) || !aligned(saturated, 4) ||
        !aligned(flag, 4))
        return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_kv_append(static_cast<const uint16_t*>(x_bf16), rows, cols, ld_x, scale, slots,
                                           cache, ld_cache, num_slots, saturated, flag,
                                           static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

size_t mx_scale_bytes(int64_t rows, int64_t k) {
    if (rows <= 0 || k <= 0 || k % 128 != 0) return 0;
    return fp8q::mx_sf_bytes(rows, k);
}

fp8q_status mx_quantize(const void* x_bf16, int64_t rows, int64_t k, int64_t ld_x, uint8_t* codes, int64_t ld_q,
                        uint8_t* scales, int32_t* nonfinite_flag, void* stream) {
    if (rows < 0 || k < 0 || ld_x < k || ld_q < k) return FP8Q_EINVAL;
    if (k % 128 != 0) return FP8Q_ESHAPE;
    if (rows == 0 || k == 0) return FP8Q_OK;
    if (x_bf16 == nullptr || codes == nullptr || scales == nullptr) return FP8Q_EINVAL;
    if (!aligned(x_bf16, 16) || ld_x % 8 != 0 || !aligned(codes, 8) || ld_q % 8 != 0 || !aligned(nonfinite_flag, 4))
        return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_mx_quantize(static_cast<const uint16_t*>(x_bf16), rows, k, ld_x, codes, ld_q, scales,
                                             nonfinite_flag, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

fp8q_status fp8_mx_gemm(const uint8_t* a, int64_t ld_a, const uint8_t* a_scales, const uint8_t* b, int64_t ld_b,
                        const uint8_t* b_scales, void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m, int64_t n,
                        int64_t k, void* stream) {
    if (m < 0 || n < 0 || k < 0 || ld_a < k || ld_b < k || ld_d < n) return FP8Q_EINVAL;
    if (d_dtype != FP8Q_OUT_BF16 && d_dtype != FP8Q_OUT_F32) return FP8Q_EINVAL;
    if (k % 128 != 0 || n % 256 != 0) return FP8Q_ESHAPE;
    if (m == 0 || n == 0) return FP8Q_OK;
    if (k == 0) return FP8Q_EUNSUPPORTED;
    if (a == nullptr || b == nullptr || a_scales == nullptr || b_scales == nullptr || d == nullptr) return FP8Q_EINVAL;
    const int esz = d_dtype == FP8Q_OUT_F32 ? 4 : 2;
    if (!aligned(a, 16) || !aligned(b, 16) || ld_a % 16 != 0 || ld_b % 16 != 0 || !aligned(a_scales, 16) ||
        !aligned(b_scales, 16) || !aligned(d, 16) || (ld_d * esz) % 16 != 0)
        return FP8Q_EALIGN;
    fp8q_status st = check_device();
    if (st != FP8Q_OK) return st;
    cudaError_t e = fp8q::launch_fp8_mx_gemm(a, ld_a, a_scales, b, ld_b, b_scales, d, ld_d, d_dtype == FP8Q_OUT_F32, m,
                                             n, k, fp8q::tensor_map_encode_fn(), static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return from_cuda(e);
}

size_t fp8_block_gemm_workspace_size(int64_t m, int64_t n, int64_t k) {
    return fp8q::gemm_workspace_bytes(m, n, k, false);
}

size_t fp8_block_gemm_grouped_workspace_size(int64_t, int64_t, int64_t, int32_t) { return 0; }

static fp8q_status gemm_common_checks(const uint8_t* a, int64_t ld_a, const float* a_scales,
                                      int64_t ld_sa, const uint8_t* b, int64_t ld_b,
                                      const float* b_scales, int64_t ld_sb, void* d, int64_t ld_d,
                                      fp8q_out_dtype d_dtype, int64_t m, int64_t n, int64_t k) {
    if (m < 0 || n < 0 || k < 0) return FP8Q_EINVAL;
    if (d_dtype != FP8Q_OUT_BF16 && d_dtype != FP8Q_OUT_F32) return FP8Q_EINVAL;
    if (ld_a < k || ld_b < k || ld_d < n || ld_sa < m || ld_sb < k / 128) return FP8Q_EINVAL;
    if (k % 128 != 0 || n % 8 != 0) return FP8Q_ESHAPE;
    if (m == 0 || n == 0) return FP8Q_OK;
    if (d == nullptr) return FP8Q_EINVAL;
    if (k == 0) return FP8Q_OK;
    if (a == nullptr || b == nullptr || a_scales == nullptr || b_scales == nullptr) return FP8Q_EINVAL;
    const int64_t esz = d_dtype == FP8Q_OUT_F32 ? 4 : 2;
    if (!aligned(a, 16) || !aligned(b, 16) || ld_a % 16 != 0 || ld_b % 16 != 0 || !aligned(d, 16) ||
        (ld_d * esz) % 16 != 0 || !aligned(a_scales, 4) || !aligned(b_scales, 4))
        return FP8Q_EALIGN;
    if (m > 0x7FFFFFFFLL || n > 0x7FFFFFFFLL || k > 0x7FFFFFFFLL) return FP8Q_EINVAL;
    return check_device();
}

static fp8q_status zero_output(void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m, int64_t n,
                               void* stream) {
    const size_t esz = d_dtype == FP8Q_OUT_F32 ? 4 : 2;
    return from_cuda(cudaMemset2DAsync(d, ld_d * esz, 0, n * esz, m, static_cast<cudaStream_t>(stream)));
}

fp8q_status fp8_block_gemm(const uint8_t* a, int64_t ld_a, const float* a_scales, int64_t ld_sa,
                           const uint8_t* b, int64_t ld_b, const float* b_scales, int64_t ld_sb,
                           void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m, int64_t n,
                           int64_t k, void* workspace, size_t workspace_bytes, void* stream) {
    if (workspace != nullptr && !aligned(workspace, 256)) return FP8Q_EALIGN;
    fp8q_status st = gemm_common_checks(a, ld_a, a_scales, ld_sa, b, ld_b, b_scales, ld_sb, d, ld_d,
                                        d_dtype, m, n, k);
    if (st != FP8Q_OK || m == 0 || n == 0) return st;
    if (k == 0) return zero_output(d, ld_d, d_dtype, m, n, stream);
    fp8q::GemmArgs g{};
    g.a = a;
    g.ld_a = ld_a;
    g.sa = a_scales;
    g.ld_sa = ld_sa;
    g.b = b;
    g.ld_b = ld_b;
    g.stride_b = 0;
    g.sb = b_scales;
    g.ld_sb = ld_sb;
    g.stride_sb = 0;
    g.d = d;
    g.ld_d = ld_d;
    g.out_f32 = d_dtype == FP8Q_OUT_F32;
    g.m = m;
    g.n = n;
    g.k = k;
    g.offsets = nullptr;
    g.groups = 1;
    g.workspace = workspace;
    g.workspace_bytes = workspace_bytes;
    int launched = 0;
    cudaError_t e = fp8q::launch_fp8_block_gemm(g, static_cast<cudaStream_t>(stream), &launched);
    g_launches.fetch_add(launched);
    return from_cuda(e);
}

// fp8_linear_dynamic: quantize_act_per_token_group into the workspace, then fp8_block_gemm;
// workspace = [GEMM split-K workspace, at least the 4 KB of counters][codes m x k][scales].
namespace {
constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
int64_t act_ld_s(int64_t m) { return (m + 3) / 4 * 4; }
// The workspace may be shared with fp8_block_gemm calls of other shapes, whose split-K counters
// (the first 4 KB, "left zeroed") must stay zero: the activation buffers start past them.
size_t act_codes_offset(int64_t m, int64_t n, int64_t k) {
    return align_up(std::max<size_t>(fp8q::gemm_workspace_bytes(m, n, k, false), 4096));
}
}  // namespace

size_t fp8_linear_dynamic_workspace_size(int64_t m, int64_t n, int64_t k) {
    if (m <= 0 || n <= 0 || k <= 0) return 0;
    return act_codes_offset(m, n, k) + align_up(static_cast<size_t>(m * k)) +
           static_cast<size_t>(k / 128) * act_ld_s(m) * 4;
}

fp8q_status fp8_linear_dynamic(const void* x_bf16, int64_t ld_x, const uint8_t* b, int64_t ld_b,
                               const float* b_scales, int64_t ld_sb, void* d, int64_t ld_d, fp8q_out_dtype d_dtype,
                               int64_t m, int64_t n, int64_t k, int32_t* nonfinite_flag, void* workspace,
                               size_t workspace_bytes, void* stream) {
    if (workspace != nullptr && !aligned(workspace, 256)) return FP8Q_EALIGN;
    if (m < 0 || n < 0 || k < 0 || ld_x < k) return FP8Q_EINVAL;
    // the GEMM's checks with the activation codes' layout (ld = k) standing in for a
    const uint8_t* fake_a = reinterpret_cast<const uint8_t*>(16);
    fp8q_status st = gemm_common_checks(fake_a, (k + 15) / 16 * 16, reinterpret_cast<const float*>(16),
                                        act_ld_s(m), b, ld_b, b_scales, ld_sb, d, ld_d, d_dtype, m, n, k);
    if (st != FP8Q_OK || m == 0 || n == 0) return st;
    if (x_bf16 == nullptr && k > 0) return FP8Q_EINVAL;
    if (k > 0 && (!aligned(x_bf16, 16) || ld_x % 8 != 0)) return FP8Q_EALIGN;
    if (nonfinite_flag != nullptr && !aligned(nonfinite_flag, 4)) return FP8Q_EALIGN;
    if (k == 0) return zero_output(d, ld_d, d_dtype, m, n, stream);
    if (workspace == nullptr || workspace_bytes < fp8_linear_dynamic_workspace_size(m, n, k)) return FP8Q_EWORKSPACE;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t gws = fp8q::gemm_workspace_bytes(m, n, k, false);
    {
        // decode sizes: the GEMM kernel quantizes the activations itself (one launch)
        fp8q::GemmArgs f{};
        f.a = nullptr;
        f.ld_a = k;
        f.sa = nullptr;
        f.ld_sa = act_ld_s(m);
        f.b = b;
        f.ld_b = ld_b;
        f.sb = b_scales;
        f.ld_sb = ld_sb;
        f.d = d;
        f.ld_d = ld_d;
        f.out_f32 = d_dtype == FP8Q_OUT_F32;
        f.m = m;
        f.n = n;
        f.k = k;
        f.groups = 1;
        f.workspace = gws > 0 ? workspace : nullptr;
        f.workspace_bytes = gws;
        f.x_bf16 = static_cast<const uint16_t*>(x_bf16);
        f.ld_x = ld_x;
        f.nonfinite_flag = nonfinite_flag;
        if (fp8q::skinny_fused_act_applies(f)) {
            int launched = 0;
            const cudaError_t ef = fp8q::launch_fp8_block_gemm(f, s, &launched);
            g_launches.fetch_add(launched);
            return from_cuda(ef);
        }
    }
    char* base = static_cast<char*>(workspace);
    const size_t off = act_codes_offset(m, n, k);
    uint8_t* codes = reinterpret_cast<uint8_t*>(base + off);
    float* scales = reinterpret_cast<float*>(base + off + align_up(static_cast<size_t>(m * k)));
    // (the quantizer is launched with programmatic dependent launch, the decode GEMM too: the
    // GEMM's weight prefetch overlaps the quantization)
    cudaError_t e = fp8q::launch_act_per_token_group(static_cast<const uint16_t*>(x_bf16), m, k, ld_x, codes, k,
                                                     scales, act_ld_s(m), nonfinite_flag, s);
    if (e != cudaSuccess) return from_cuda(e);
    g_launches.fetch_add(1);
    fp8q::GemmArgs g{};
    g.a = codes;
    g.ld_a = k;
    g.sa = scales;
    g.ld_sa = act_ld_s(m);
    g.b = b;
    g.ld_b = ld_b;
    g.sb = b_scales;
    g.ld_sb = ld_sb;
    g.d = d;
    g.ld_d = ld_d;
    g.out_f32 = d_dtype == FP8Q_OUT_F32;
    g.m = m;
    g.n = n;
    g.k = k;
    g.groups = 1;
    g.workspace = gws > 0 ? workspace : nullptr;
    g.workspace_bytes = gws;
    int launched = 0;
    e = fp8q::launch_fp8_block_gemm(g, s, &launched);
    g_launches.fetch_add(launched);
    return from_cuda(e);
}

fp8q_status fp8_block_gemm_grouped(const uint8_t* a, int64_t ld_a, const float* a_scales,
                                   int64_t ld_sa, const uint8_t* b, int64_t ld_b, int64_t stride_b,
                                   const float* b_scales, int64_t ld_sb, int64_t stride_sb,
                                   void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m_total,
                                   int64_t n, int64_t k, const int32_t* offsets_dev,
                                   int32_t num_groups, void* workspace, size_t workspace_bytes,
                                   void* stream) {
    (void)workspace;
    (void)workspace_bytes;
    if (num_groups < 0) return FP8Q_ESHAPE;
    fp8q_status st = gemm_common_checks(a, ld_a, a_scales, ld_sa, b, ld_b, b_scales, ld_sb, d, ld_d,
                                        d_dtype, m_total, n, k);
    if (st != FP8Q_OK || m_total == 0 || n == 0 || num_groups == 0) return st;
    if (offsets_dev == nullptr) return FP8Q_EINVAL;
    if (!aligned(offsets_dev, 4)) return FP8Q_EALIGN;
    if (num_groups > 1 && (stride_b < ld_b * n || stride_sb < ((n + 127) / 128) * ld_sb))
        return FP8Q_EINVAL;
    if (stride_b % 16 != 0) return FP8Q_EALIGN;
    if (k == 0) return zero_output(d, ld_d, d_dtype, m_total, n, stream);
    fp8q::GemmArgs g{};
    g.a = a;
    g.ld_a = ld_a;
    g.sa = a_scales;
    g.ld_sa = ld_sa;
    g.b = b;
    g.ld_b = ld_b;
    g.stride_b = stride_b;
    g.sb = b_scales;
    g.ld_sb = ld_sb;
    g.stride_sb = stride_sb;
    g.d = d;
    g.ld_d = ld_d;
    g.out_f32 = d_dtype == FP8Q_OUT_F32;
    g.m = m_total;
    g.n = n;
    g.k = k;
    g.offsets = offsets_dev;
    g.groups = num_groups;
    g.workspace = nullptr;
    g.workspace_bytes = 0;
    int launched = 0;
    cudaError_t e = fp8q::launch_fp8_block_gemm(g, static_cast<cudaStream_t>(stream), &launched);
    g_launches.fetch_add(launched);
    return from_cuda(e);
}

}  // extern "C"

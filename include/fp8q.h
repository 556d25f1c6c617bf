/*
 * fp8q.h -- C-ABI of libfp8q, the B200 (sm_100a) hot path of the FP8 W8A8 rollout in
 * "FP8-RL: A Practical and Stable Low-Precision Stack for LLM Reinforcement Learning"
 * (arXiv 2601.18150).  PAPER.md = /root/reference/PAPER.md (line numbers cited).
 *
 * The three operations of the paper's statement of the problem (§2.1):
 *   quantize_weight_blockwise      Eq. (1): W_hat = round(W / scale), one
 *                                  scale per 128x128 block from the block's max |W|; done at
 *                                  every weight synchronisation.
 *   quantize_act_per_token_group   dynamic activation quantization, one
 *                                  scale per token per 128 channels (1x128).
 *   fp8_block_gemm[_grouped]       the W8A8 linear / MoE expert GEMM consuming both
 *                                  (PAPER.md:62,99,129,147), blockwise scales promoted per
 *                                  128-deep k-block into an fp32 accumulator.
 *
 * Arithmetic (readings fixed in DESIGN.md §3; Q-numbers from SURVEY.md §8(c)):
 *   E4M3 = OCP E4M3FN (bias 7, no Inf, NaN = S.1111.111, max 448)          (Q9)
 *   amax  = max |x| over the block/group's in-bounds elements (BF16 widened exactly)
 *   s     = RN32(amax / 448)  (one IEEE binary32 division); amax == 0 -> s = 1    (Q2,Q4,Q5)
 *   code  = E4M3_RNE_satfinite(RN32(x / s)); the sign of zero is kept (-0 -> 0x80) (Q1,Q3,Q6,Q7)
 *   GEMM  D[m,n] = sum_kb (sa[kb][m] * sb[n/128][kb]) * P_kb[m,n],
 *         P_kb[m,n] = sum_{k in kb} dec(a[m,k]) dec(b[n,k])   (fp32 tensor-core partials,
 *         fp32 promotion in k-block order, deterministic; BF16 output = RNE of the F32 result)
 *
 * Conventions (all entry points):
 *   - Ownership: the caller owns every buffer; the library never allocates device memory.
 *     All data pointers are DEVICE pointers unless stated otherwise.
 *   - Asynchrony: work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and the call returns immediately.
 *   - Validation errors are synchronous: a non-OK status means nothing was enqueued and no
 *     output was touched.  Device faults surface at the next synchronisation as cudaError.
 *   - Stateless apart from once-per-process kernel attributes and a cached driver entry
 *     point; thread-safe.  No C++ exception crosses the ABI.
 *   - Deterministic: identical inputs give bitwise-identical outputs (no float atomics).
 *   - Layouts are row-major with an explicit leading dimension in ELEMENTS.
 */
#ifndef FP8Q_H_
#define FP8Q_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FP8Q_OK = 0,
    FP8Q_EINVAL = 1,       /* null pointer with non-empty extent, negative dim, ld < extent */
    FP8Q_ESHAPE = 2,       /* k % 128 (act, GEMM), k % 8 (weights), n % 8 (GEMM), bad groups */
    FP8Q_EALIGN = 3,       /* pointer / leading-dimension alignment required by vector IO/TMA */
    FP8Q_ECUDA = 4,        /* a CUDA runtime call failed at enqueue time */
    FP8Q_EUNSUPPORTED = 5, /* device is not sm_100 or a feature is not built */
    FP8Q_EWORKSPACE = 6    /* workspace smaller than *_workspace_size() */
} fp8q_status;

typedef enum { FP8Q_OUT_BF16 = 0, FP8Q_OUT_F32 = 1 } fp8q_out_dtype;

/* Human-readable name of a status code (static storage; never NULL). */
const char* fp8q_status_string(fp8q_status s);
/* The CUDA runtime's message for the last cudaError behind an FP8Q_ECUDA returned on this thread
 * ("no error" if none): diagnostics only. */
const char* fp8q_last_cuda_error(void);

/* Library ABI version (major*10000 + minor*100 + patch). */
int32_t fp8q_version(void);

/*
 * quantize_weight_blockwise -- PAPER.md:54-58 (§2.1.1, Eq. (1)); per-step resync PAPER.md:72.
 *   w_bf16  [n, k] BF16, row stride ld_w (elements).  nn.Linear layout [out = N, in = K].
 *   codes   [n, k] E4M3 bytes out, row stride ld_q.
 *   scales  [ceil(n/128), ceil(k/128)] fp32 out, row stride ld_s >= ceil(k/128).
 *           Block (i, j) covers rows [128i, min(128i+128, n)) x cols [128j, min(128j+128, k));
 *           ragged edge blocks are clipped (their amax is over in-bounds elements only).
 *   nonfinite_flag  nullable device int32; set to 1 (never cleared) if any input element is
 *           NaN/Inf.  The codes/scales of such a block are then unspecified (the oracle
 *           rejects such input).
 *   Requirements: n, k >= 0; ld_w >= k, ld_q >= k; k % 8 == 0 (else ESHAPE);
 *     w_bf16 16-byte aligned, ld_w % 8 == 0; codes 8-byte aligned, ld_q % 8 == 0 (else EALIGN).
 *   Work: 3 + 4/16384 bytes of HBM traffic per element (2 read, 1 written, 4 per block).
 */
fp8q_status quantize_weight_blockwise(const void* w_bf16, int64_t n, int64_t k, int64_t ld_w,
                                      uint8_t* codes, int64_t ld_q, float* scales, int64_t ld_s,
                                      int32_t* nonfinite_flag, void* stream);

/*
 * quantize_weight_blockwise_batched -- the per-step weight synchronisation of PAPER.md:72
 * re-quantizes every in-scope linear weight; this entry point does exactly what `count`
 * quantize_weight_blockwise calls would do, but in as few kernel launches as possible (up to
 * 16 tensors per launch), so small tensors do not each pay a launch and a pipeline ramp.
 *   tensors  HOST array of `count` descriptors (read during the call only); the pointers in
 *            them are device pointers with the meaning and requirements of
 *            quantize_weight_blockwise.  Every descriptor is validated before anything is
 *            enqueued; the first failing one determines the status.
 *   nonfinite_flag, stream  as quantize_weight_blockwise (one flag for the whole batch).
 */
typedef struct {
    const void* w_bf16;
    int64_t n, k, ld_w;
    uint8_t* codes;
    int64_t ld_q;
    float* scales;
    int64_t ld_s;
} fp8q_weight_tensor;

fp8q_status quantize_weight_blockwise_batched(const fp8q_weight_tensor* tensors, int32_t count,
                                              int32_t* nonfinite_flag, void* stream);

/*
 * quantize_weight_blockwise_fanout -- SURVEY §8(f) NEXT-1: the per-step requant of a rank's
 *   shard written straight into EVERY rank's engine buffer, so no separate all-gather pass
 *   re-reads the codes ("retrieved ... quantized ... loaded").  Same element map
 *   as quantize_weight_blockwise_batched; each code / scale store goes to
 *       tensors[i].codes + codes_delta[d]   and   tensors[i].scales + scales_delta[d] (bytes)
 *   for d in [0, num_dest): peer-mapped buffers of identical layout (e.g. torch symmetric
 *   memory: delta = peer base - local base; include delta 0 for the local copy).  Over
 *   NVLink/NVSwitch the stores are P2P writes issued by the quantizer itself.  The caller
 *   orders the peers' reads after the launch (e.g. a barrier on the symmetric-memory handle).
 *   Requirements: 1 <= num_dest <= 8 (EINVAL); codes_delta % 16 == 0, scales_delta % 4 == 0
 *   (EALIGN); every tensor on the wide path: k % 16 == 0, w 32-byte aligned, ld_w % 16 == 0,
 *   codes 16-byte aligned, ld_q % 16 == 0 (EUNSUPPORTED otherwise); the rest as
 *   quantize_weight_blockwise.
 */
fp8q_status quantize_weight_blockwise_fanout(const fp8q_weight_tensor* tensors, int32_t count, int32_t num_dest,
                                             const int64_t* codes_delta, const int64_t* scales_delta,
                                             int32_t* nonfinite_flag, void* stream);

/*
 * quantize_act_per_token_group -- dynamic activation quantization, PAPER.md:46,65,73;
 * granularity 1x128 (per token m, per 128-channel group g).
 *   x_bf16  [m, k] BF16, row stride ld_x.
 *   codes   [m, k] E4M3 bytes out, row stride ld_q.
 *   scales  fp32 out, MN-MAJOR: the scale of (m, g) is scales[g * ld_s + m]; ld_s >= m and
 *           ld_s % 4 == 0 so every group's column of M scales is a 16-byte aligned row
 *           (the layout fp8_block_gemm consumes as `a_scales`).
 *   nonfinite_flag  as above.
 *   Requirements: k % 128 == 0 (ESHAPE); x_bf16 16-byte aligned, ld_x % 8 == 0, codes 8-byte
 *     aligned, ld_q % 8 == 0, scales 4-byte aligned, ld_s % 4 == 0 (EALIGN).
 *   Work: 3 + 4/128 bytes of HBM traffic per element.
 */
fp8q_status quantize_act_per_token_group(const void* x_bf16, int64_t m, int64_t k, int64_t ld_x,
                                         uint8_t* codes, int64_t ld_q, float* scales, int64_t ld_s,
                                         int32_t* nonfinite_flag, void* stream);

/*
 * quantize_act_per_token_group_batched -- the activation quantizations of one forward step
 * (every linear layer's input is quantized dynamically) issued together: does
 * exactly what `count` quantize_act_per_token_group calls would do, but in as few kernel
 * launches as possible (up to 8 tensors per persistent launch), so the inputs of a layer's
 * GEMMs share one pipeline ramp and one tail.
 *   tensors  HOST array of `count` descriptors (read during the call only); the pointers in
 *            them are device pointers with the meaning and requirements of
 *            quantize_act_per_token_group.  Every descriptor is validated before anything is
 *            enqueued; the first failing one determines the status.
 *   nonfinite_flag, stream  as quantize_act_per_token_group (one flag for the whole batch).
 */
typedef struct {
    const void* x_bf16;
    int64_t m, k, ld_x;
    uint8_t* codes;
    int64_t ld_q;
    float* scales;
    int64_t ld_s;
} fp8q_act_tensor;

fp8q_status quantize_act_per_token_group_batched(const fp8q_act_tensor* tensors, int32_t count,
                                                 int32_t* nonfinite_flag, void* stream);

/*
 * rmsnorm_quantize_act_per_token_group -- SURVEY §8(f) NEXT-2: quantize_act_per_token_group
 * fused into its producer on the rollout forward (the RMSNorm before q/k/v and gate/up):
 *   y[m, j] = BF16_RNE( x[m, j] / sqrt(mean_i x[m, i]^2 + eps) * gamma[j] )   (binary32 inside)
 *   codes, scales = quantize_act_per_token_group(y)  (identical element map and layouts)
 * y never reaches HBM unless y_bf16 (nullable, row stride ld_y) is given.
 *   Requirements: k % 128 == 0 and k <= 4096 (one token row per warp, held in registers;
 *     Qwen3 hidden sizes are 4096 / 2048) (ESHAPE); x, gamma 16-byte aligned, ld_x % 8 == 0,
 *     codes 8-byte aligned, ld_q % 8 == 0, scales as quantize_act_per_token_group, y_bf16
 *     16-byte aligned with ld_y % 8 == 0 (EALIGN).
 */
fp8q_status rmsnorm_quantize_act_per_token_group(const void* x_bf16, const void* gamma_bf16, float eps,
                                                 int64_t m, int64_t k, int64_t ld_x, uint8_t* codes,
                                                 int64_t ld_q, float* scales, int64_t ld_s, void* y_bf16,
                                                 int64_t ld_y, int32_t* nonfinite_flag, void* stream);

/*
 * silu_mul_quantize_act_per_token_group -- NEXT-2 for the down_proj input:
 *   gate = gate_up[:, 0:inter], up = gate_up[:, inter:2*inter]   (row stride ld_gu)
 *   y = BF16_RNE( gate / (1 + exp(-gate)) * up )   (binary32 inside), then quantized as above.
 *   Requirements: inter % 128 == 0 (ESHAPE); alignment as rmsnorm_quantize_act_per_token_group.
 */
fp8q_status silu_mul_quantize_act_per_token_group(const void* gate_up_bf16, int64_t m, int64_t inter,
                                                  int64_t ld_gu, uint8_t* codes, int64_t ld_q, float* scales,
                                                  int64_t ld_s, void* y_bf16, int64_t ld_y,
                                                  int32_t* nonfinite_flag, void* stream);

/*
 * fp8_block_gemm -- the W8A8 linear Y = X W^T, blockwise scales promoted
 * per 128-deep k-block (DeepSeek-V3 granularity cited at PAPER.md:233):
 *   D[m,n] = sum_kb sa[kb][m] * sb[n/128][kb] * sum_{k in kb} dec(a[m,k]) * dec(b[n,k])
 *   a        [m, k] E4M3 codes (K-major), row stride ld_a bytes.
 *   a_scales MN-major [k/128][ld_sa] fp32 (as written by quantize_act_per_token_group).
 *   b        [n, k] E4M3 codes (K-major, nn.Linear weight), row stride ld_b bytes.
 *   b_scales [ceil(n/128)][ld_sb] fp32 (as written by quantize_weight_blockwise), ld_sb >= k/128.
 *   d        [m, n] out, BF16 or F32 per d_dtype, row stride ld_d elements.
 *   workspace / workspace_bytes: optional (NULL / 0 allowed).  With at least
 *           fp8_block_gemm_workspace_size(m, n, k) bytes (256-byte aligned, ZERO-FILLED before
 *           its first use; every launch leaves it zeroed again), small-M problems (decode,
 *           M <= 128) whose weight has many 128-row tiles split the K loop over more CTAs
 *           (stream-K), and the tile kernels split the K loop of the tiles of their last,
 *           partial wave (the "tail": T mod U tiles, U = SMs or CTA pairs) into slices:
 *           slices park fp32 partials in the workspace and the last slice of each tile sums
 *           them in slice order (deterministic).  Without it the same problem runs unsplit
 *           (slower, equal up to fp32 summation order).  A workspace must not be shared by concurrently
 *           running GEMMs.  Weights with few tiles (tiles <= SMs / 2) split K inside a thread-
 *           block cluster instead (partials reduced in CTA-rank order through distributed
 *           shared memory) and never touch the workspace.
 *   Kernels: 1 <= m <= 128 with 16-byte-aligned a_scales and ld_sa % 4 == 0 runs the swap-AB
 *     decode kernel (weight rows in the MMA M dimension, tokens in N), and so does
 *     129 <= m <= 256 where its cluster split-K applies and the CTA pair would not split its
 *     tiles along K over most SMs; otherwise the 128 x 256 / 256 x 256 (CTA pair) tile kernel.  All compute the same per-k-block promotion in the same k order
 *     (split-K partial sums are added in a fixed order: results are deterministic).
 *   Requirements: k % 128 == 0, n % 8 == 0 (ESHAPE); a, b 16-byte aligned with ld_a % 16 ==
 *     0 and ld_b % 16 == 0 (TMA); d 16-byte aligned with ld_d * sizeof(out) % 16 == 0;
 *     a_scales/b_scales 4-byte aligned (EALIGN).  m == 0 or n == 0 is a no-op; k == 0 writes 0.
 *   Work: 2*m*n*k FLOP on the tensor cores (kind::f8f6f4), m*n*k/128 fp32 promotion FMAs.
 */
size_t fp8_block_gemm_workspace_size(int64_t m, int64_t n, int64_t k); /* 0: never splits */
fp8q_status fp8_block_gemm(const uint8_t* a, int64_t ld_a, const float* a_scales, int64_t ld_sa,
                           const uint8_t* b, int64_t ld_b, const float* b_scales, int64_t ld_sb,
                           void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m, int64_t n,
                           int64_t k, void* workspace, size_t workspace_bytes, void* stream);

/*
 * fp8_linear_dynamic -- one W8A8 linear layer of the rollout forward as the engine calls it:
 * the BF16 layer input quantized dynamically per token per 128 channels (the
 * 1x128 granularity of PAPER.md:233) and multiplied by the blockwise-quantized weight
 * (PAPER.md:99,129).  Result bit-identical to quantize_act_per_token_group(x) followed by
 * fp8_block_gemm(codes, scales, b, b_scales) -- the same element map and the same GEMM.
 *   x_bf16   [m, k] BF16 activations, row stride ld_x (16-byte aligned, ld_x % 8 == 0).
 *   b, b_scales, d, d_dtype, m, n, k   as fp8_block_gemm.
 *   nonfinite_flag  as quantize_act_per_token_group (set if x holds NaN/Inf; nullable).
 *   workspace / workspace_bytes: at least fp8_linear_dynamic_workspace_size(m, n, k) bytes,
 *     256-byte aligned, ZERO-FILLED before first use (the GEMM's split-K counters; every launch
 *     leaves them zeroed), holding the activation codes and scales between the two kernels
 *     (FP8Q_EWORKSPACE if missing or too small).  At m <= 16 where the decode kernel applies
 *     (and its CTAs' activation k-blocks fit 32 shared-memory slots: every Qwen3-8B linear), ONE
 *     launch: the decode GEMM's promotion warps quantize the BF16 rows of the CTA's k-blocks into
 *     shared memory after griddepcontrol.wait, with the quantizers' element map (the codes and
 *     scales never reach the workspace).  Otherwise the quantizer is launched with programmatic
 *     dependent launch and, for <= 256 tokens, as a shared-memory-free kernel, so the decode
 *     GEMM's weight prefetch overlaps it.  (round 2's single-kernel form, which
 *     quantized per k-block through the ring, was slower than the pair and removed.)
 *   Requirements as fp8_block_gemm (k % 128, n % 8, alignments).
 */
size_t fp8_linear_dynamic_workspace_size(int64_t m, int64_t n, int64_t k);
fp8q_status fp8_linear_dynamic(const void* x_bf16, int64_t ld_x, const uint8_t* b, int64_t ld_b,
                               const float* b_scales, int64_t ld_sb, void* d, int64_t ld_d, fp8q_out_dtype d_dtype,
                               int64_t m, int64_t n, int64_t k, int32_t* nonfinite_flag, void* workspace,
                               size_t workspace_bytes, void* stream);

/*
 * fp8_block_gemm_grouped -- MoE expert layers in FP8 ("MoE expert layers
 * (fc1, fc2)").  Group g multiplies A rows [offsets[g], offsets[g+1]) by
 * B_g = b + g * stride_b (bytes) with scales b_scales + g * stride_sb (elements):
 *   D[r, n] = fp8_block_gemm(A[r,:], B_g)[n]   for offsets[g] <= r < offsets[g+1].
 *   offsets_dev  DEVICE int32 [num_groups + 1], offsets[0] = 0, non-decreasing,
 *                offsets[num_groups] = m_total (the router output stays on the device; no
 *                host sync).  Violating the precondition is undefined behaviour.
 *   a_scales     MN-major [k/128][ld_sa] over all m_total rows.
 *   Requirements as fp8_block_gemm, plus stride_b % 16 == 0, num_groups >= 0.
 */
size_t fp8_block_gemm_grouped_workspace_size(int64_t m_total, int64_t n, int64_t k,
                                             int32_t num_groups);
fp8q_status fp8_block_gemm_grouped(const uint8_t* a, int64_t ld_a, const float* a_scales,
                                   int64_t ld_sa, const uint8_t* b, int64_t ld_b, int64_t stride_b,
                                   const float* b_scales, int64_t ld_sb, int64_t stride_sb,
                                   void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m_total,
                                   int64_t n, int64_t k, const int32_t* offsets_dev,
                                   int32_t num_groups, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* ------------------------------------------------------------------------------------------
 * NEXT-3: FP8 KV cache with per-step scale recalibration (§2.3.1:
 * "we trigger a forced recalibration ... before the rollout phase of each RL step" (inference
 * side) / "recalibrates QKV scales using the updated policy weights and a subset of training
 * data" (trainer side)).  One scalar scale per layer and tensor (K, V, Q):
 *   calibration   amax = max |x| over every calibration element (all batches),
 *                 scale = RN32(amax / 448), amax == 0 -> 1            (readings K1, Q4, Q5)
 *   append        cache[slot[r]][c] = E4M3_RNE_sat(RN32(x[r][c] / scale))   (K2, K4; O5)
 *   saturation    an element saturates iff |RN32(x / scale)| >= 464 (its code is then +-448);
 *                 such elements are counted                                    (K3)
 * Layout: x is BF16 [rows = tokens, cols = heads * head_dim] with row stride ld_x elements;
 * the cache is uint8 [num_slots][ld_cache].  All pointers are device pointers owned by the
 * caller; everything is enqueued on `stream`; no host sync.
 * ------------------------------------------------------------------------------------------ */

/*
 * kv_amax_update -- *amax_bits = max(*amax_bits, BF16 bits of max |x|) (sign-cleared BF16 bits
 *   in a uint32; the caller zeroes it to start a calibration = "reset calculate_kv_scales").
 *   Deterministic (an integer max).  flag (nullable): bit 0 set if x holds NaN/Inf.
 *   Errors: negative sizes or ld_x < cols (EINVAL); misaligned pointers (EALIGN).
 */
fp8q_status kv_amax_update(const void* x_bf16, int64_t rows, int64_t cols, int64_t ld_x, uint32_t* amax_bits,
                           int32_t* flag, void* stream);

/*
 * kv_scale_from_amax -- scales[i] = RN32(amax_i / 448) (amax_i == 0 -> 1) for count layers /
 *   tensors at once; amax_bits as written by kv_amax_update.
 */
fp8q_status kv_scale_from_amax(const uint32_t* amax_bits, int64_t count, float* scales, void* stream);

/*
 * kv_quantize_append -- writes the E4M3 codes of x's rows into cache rows slots[r] (slots
 *   nullable: row r -> cache row r, then rows <= num_slots is required (ESHAPE)), with the
 *   scalar *scale (device).  saturated (nullable): += number of saturated elements.  flag
 *   (nullable): |= 1 if x holds NaN/Inf (those codes unspecified), |= 2 if a slot is outside
 *   [0, num_slots) (that row is skipped).  Rows must not map to the same slot twice.
 *   Errors: EINVAL (sizes, ld_x < cols, ld_cache < cols, null x/scale/cache), EALIGN.
 *   Traffic: 2 B read + 1 B written per element (HBM-bound).
 */
fp8q_status kv_quantize_append(const void* x_bf16, int64_t rows, int64_t cols, int64_t ld_x, const float* scale,
                               const int32_t* slots, uint8_t* cache, int64_t ld_cache, int64_t num_slots,
                               uint32_t* saturated, int32_t* flag, void* stream);

/* ------------------------------------------------------------------------------------------
 * NEXT-4: MXFP8 variant (PAPER.md:235 names Blackwell FP8 support).  NOT
 * the paper's quantizer: power-of-two E8M0 scales on 1x32 blocks along K, so the tcgen05
 * block-scaled MMA applies them in hardware (readings X1-X3):
 *   e = the smallest integer >= -127 with 448 * 2^e >= amax(block) (amax == 0 -> 0),
 *   code = E4M3_RNE(x / 2^e) (exact division: no element ever saturates), scale byte = e + 127.
 * Scale layout ("native"): byte (row r, 32-K sub-block j) at
 *   ((r / 128) * (k / 128) + j / 4) * 512 + (r % 128) * 4 + j % 4,
 * i.e. one contiguous 512-byte chunk per (128-row block, 128-deep k-block);
 * mx_scale_bytes(rows, k) = ceil(rows / 128) * (k / 128) * 512.
 * ------------------------------------------------------------------------------------------ */
size_t mx_scale_bytes(int64_t rows, int64_t k); /* 0 for invalid sizes */

/*
 * mx_quantize -- BF16 [rows, k] (row stride ld_x) -> codes [rows, k] (row stride ld_q) and
 *   native scale bytes (mx_scale_bytes(rows, k) bytes, caller-allocated).  Works for either
 *   operand (activations: rows = tokens; weights: rows = output features).
 *   Requirements: k % 128 == 0 (ESHAPE); x 16-byte aligned, ld_x % 8 == 0, codes 8-byte
 *   aligned, ld_q % 8 == 0 (EALIGN).  nonfinite_flag as quantize_weight_blockwise.
 */
fp8q_status mx_quantize(const void* x_bf16, int64_t rows, int64_t k, int64_t ld_x, uint8_t* codes, int64_t ld_q,
                        uint8_t* scales, int32_t* nonfinite_flag, void* stream);

/*
 * fp8_mx_gemm -- D[m,n] = sum_k dec(a[m,k]) 2^(sa[m,k/32]-127) dec(b[n,k]) 2^(sb[n,k/32]-127)
 *   on the tensor cores (kind::mxf8f6f4.block_scale, fp32 accumulation in TMEM over all of K).
 *   a [m, k], b [n, k] E4M3 codes (K-major), a_scales / b_scales native E8M0 bytes from
 *   mx_quantize, d [m, n] BF16 or F32 (row stride ld_d elements).
 *   Requirements: k % 128 == 0, k > 0, n % 256 == 0 (ESHAPE / EUNSUPPORTED); a, b, scales,
 *   d 16-byte aligned, ld_a % 16 == 0, ld_b % 16 == 0, ld_d * sizeof(out) % 16 == 0 (EALIGN).
 */
fp8q_status fp8_mx_gemm(const uint8_t* a, int64_t ld_a, const uint8_t* a_scales, const uint8_t* b, int64_t ld_b,
                        const uint8_t* b_scales, void* d, int64_t ld_d, fp8q_out_dtype d_dtype, int64_t m, int64_t n,
                        int64_t k, void* stream);

/*
 * e4m3_encode_f32 -- the element encode of every quantizer above (step a3, Eq. (1)
 *   "round", readings Q1/Q7/Q9): codes[i] = E4M3_RNE_satfinite(x[i]) through the same
 *   hardware `cvt.rn.satfinite.e4m3x2.f32` instruction and the same device helper the
 *   quantizers use, applied to raw fp32 values (no scale).  Exposed so the encode can be
 *   checked against the oracle on all 2^32 fp32 bit patterns (SURVEY §8(c) O2 pin (iv)).
 *   x [n] fp32, codes [n] bytes out (device).  n >= 0; n > 0 requires x 8-byte and codes
 *   2-byte aligned and n % 2 == 0 (EALIGN / ESHAPE).  NaN input gives a NaN code.
 */
fp8q_status e4m3_encode_f32(const float* x, int64_t n, uint8_t* codes, void* stream);

/*
 * fp8q_kernel_launches -- number of kernels this library has launched in this process
 * (monotone counter; used by bench.py to report `gpu_launches`).
 */
int64_t fp8q_kernel_launches(void);


#ifdef __cplusplus
}
#endif
#endif /* FP8Q_H_ */

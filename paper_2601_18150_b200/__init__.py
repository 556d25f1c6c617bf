"""paper_2601_18150_b200 -- B200-native (sm_100a) hot path of the FP8 W8A8 rollout of
"FP8-RL: A Practical and Stable Low-Precision Stack for LLM Reinforcement Learning"
(arXiv 2601.18150): per-step blockwise weight requantization, dynamic per-token-group
activation quantization, and the blockwise-scaled FP8 GEMM (dense + grouped MoE), behind
the C-ABI in include/fp8q.h, plus the sharded weight-sync orchestration.
"""
from .fp8q import (  # noqa: F401
    Fp8qError,
    act_scales_ld,
    fp8_block_gemm,
    fp8_block_gemm_grouped,
    fp8_linear_dynamic,
    fp8_mx_gemm,
    kernel_launches,
    mx_quantize,
    mx_scales_logical,
    kv_amax_update,
    kv_quantize_append,
    kv_scale_from_amax,
    load_library,
    quantize_act_per_token_group,
    quantize_act_per_token_group_batched,
    quantize_weight_blockwise,
    quantize_weight_blockwise_batched,
    rmsnorm_quantize_act_per_token_group,
    silu_mul_quantize_act_per_token_group,
    version,
)

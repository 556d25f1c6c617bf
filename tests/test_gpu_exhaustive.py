"""Exhaustive bit-exactness of the quantizer element map on the GPU (SURVEY §0 finding 2).

Every positive finite BF16 amax A (32,639 values) paired with every BF16 x in {0} U (0, A]
-- 532,701,119 (x, amax) pairs -- packed into real 128x128 weight blocks (48,896 blocks) and
into real 1x128 activation groups (4,210,688 groups), each with both signs (so +-0 and every
negative pair too), goes through the production kernels and is compared byte for byte with
the oracle.  This is also the proof, on the hardware, that the quantizers' guarded Markstein
quotient (r = RN(1/s), q = fma-corrected x*r) gives the IEEE-division codes.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import act_scales_logical, to_dev_bf16, to_host_f32, to_host_u8

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("negate", [False, True])
def test_exhaustive_weight_map(negate):
    blocks = 0
    for chunk in synth.exhaustive_weight_chunks(blocks_per_chunk=4096, negate=negate):
        w = to_dev_bf16(chunk)
        codes, scales = fp8q.quantize_weight_blockwise(w)
        oc, os_ = oracle.quantize_weight_blockwise(chunk)
        gs = to_host_f32(scales)
        assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32)), f"scales differ in chunk at block {blocks}"
        gc = to_host_u8(codes)
        bad = np.nonzero(gc != oc)
        assert bad[0].size == 0, (f"{bad[0].size} mismatches; first at row {bad[0][0]} col {bad[1][0]}: "
                                  f"x bits {chunk[bad[0][0], bad[1][0]]:#06x} got {gc[bad][0]:#04x} want {oc[bad][0]:#04x}")
        # the block-amax element (position (0,0) of every block) always encodes to +-448
        amax_codes = gc[::128, 0]
        assert np.all(amax_codes == (0xFE if negate else 0x7E))
        blocks += chunk.shape[0] // 128
    assert blocks == synth.exhaustive_weight_num_blocks() == 48_896


@pytest.mark.parametrize("negate", [False, True])
def test_exhaustive_activation_map(negate):
    groups = 0
    k = 1024
    for chunk in synth.exhaustive_act_chunks(rows_per_chunk=1 << 16, k=k, negate=negate):
        m = chunk.shape[0]
        x = to_dev_bf16(chunk)
        codes, scales = fp8q.quantize_act_per_token_group(x)
        oc, os_ = oracle.quantize_act_per_token_group(chunk)
        gs = act_scales_logical(scales, m)
        assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32))
        gc = to_host_u8(codes)
        assert np.count_nonzero(gc != oc) == 0
        groups += m * (k // 128)
    assert groups >= synth.exhaustive_act_num_rows()

"""The seeded generators: determinism and the exhaustive (x, amax) map's coverage
(SURVEY.md §0 finding 2: 32,639 amax values, 532,701,119 pairs)."""
import numpy as np

import synth


def test_generators_deterministic():
    assert np.array_equal(synth.qwen3_weight(64, 128, 3), synth.qwen3_weight(64, 128, 3))
    assert not np.array_equal(synth.qwen3_weight(64, 128, 3), synth.qwen3_weight(64, 128, 4))
    assert np.array_equal(synth.qwen3_activation(8, 256, 1), synth.qwen3_activation(8, 256, 1))


def test_exhaustive_map_coverage():
    assert synth.exhaustive_pairs_count() == 532_701_119
    for unit in (128 * 128, 128):
        amax, start = synth._exhaustive_plan(unit)
        per = unit - 1
        covered = np.minimum(start + per, amax + 1) - start
        tot = np.bincount(amax - synth.AMAX_BITS_MIN, weights=covered)
        assert np.array_equal(tot, np.arange(synth.AMAX_BITS_MIN, synth.AMAX_BITS_MAX + 1) + 1)
    assert synth.exhaustive_weight_num_blocks() == 48_896
    first = next(synth.exhaustive_weight_chunks(blocks_per_chunk=3))
    assert first.shape == (384, 128)
    assert first[0, 0] == 1 and first[0, 1] == 0 and first[0, 2] == 1  # A=1: x in {0, 1}
    neg = next(synth.exhaustive_weight_chunks(blocks_per_chunk=1, negate=True))
    assert np.all(neg >> 15 == 1)
    rows = next(synth.exhaustive_act_chunks(rows_per_chunk=2, k=256))
    assert rows.shape == (2, 256)


def test_moe_sizes():
    s = synth.moe_group_sizes(8192, seed=0)
    assert s.sum() == 8192 * 8 and s.size == 128
    z = synth.moe_group_sizes(8192, seed=0, skew=1.2)
    assert z.sum() == 8192 * 8 and z.max() > s.max()

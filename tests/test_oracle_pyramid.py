"""Pins of the f3 literal image-pyramid mode of the oracle (stats_mode = PYRAMID, A32): levels
are rounded box means of the next finer level, block colour data are area x level
value, S_1 comes from the coarsest level, sums are then reused (Eq. 8)."""
import numpy as np
import pytest

import oracle
import synth


def stage0_sums(img, stages, M, mode):
    H, W = img.shape[:2]
    p = synth.Params(M, stages, 1, synth.lambda_pos_default(H, W, M), stats_mode=mode)
    return oracle.segment(img[None], p, stop=(oracle.STOP_STAGE_START, 0, 0, 0), map_cap=4 * H * W).sp


def test_rounding_chain_hand_worked():
    # 4x4, stages 4, 2, 1, one superpixel.  Red of the four 2x2 blocks: [1,0,0,0] -> mean 1/4
    # -> 0; [1,1,0,0] -> 1/2 -> 1 (half up); [1,1,1,0] -> 3/4 -> 1; [0,0,0,0] -> 0.  The 4x4
    # level: rhu((0 + 4 + 4 + 0) / 16) = rhu(1/2) = 1, so S_1 red = 16 x 1 = 16 (exact: 6).
    img = np.zeros((4, 4, 3), np.uint8)
    img[0:2, 0:2, 0] = [[1, 0], [0, 0]]
    img[0:2, 2:4, 0] = [[1, 1], [0, 0]]
    img[2:4, 0:2, 0] = [[1, 1], [1, 0]]
    lit = stage0_sums(img, [4, 2, 1], 1, synth.STATS_PYRAMID)
    ex = stage0_sums(img, [4, 2, 1], 1, synth.STATS_REUSE)
    assert int(lit["sum_r"][0]) == 16 and int(ex["sum_r"][0]) == 6
    assert int(lit["n"][0]) == int(ex["n"][0]) == 16
    assert int(lit["sum_x"][0]) == int(ex["sum_x"][0]) == 4 * (0 + 1 + 2 + 3)  # positions exact


def test_constant_levels_equal_exact_mode():
    # every level of a piecewise-constant image (constant on the coarsest blocks) is exact:
    # the literal pyramid changes nothing (SPEC: constant image invariant under the mean)
    rng = np.random.default_rng(3)
    coarse = rng.integers(0, 256, (4, 6, 3)).astype(np.uint8)
    img = np.repeat(np.repeat(coarse, 8, axis=0), 8, axis=1)
    p = synth.Params(6, [8, 4, 2, 1], 3, synth.lambda_pos_default(32, 48, 6))
    a = oracle.segment(img[None], p)
    p.stats_mode = synth.STATS_PYRAMID
    b = oracle.segment(img[None], p)
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.sp["sum_r"], b.sp["sum_r"]) and np.array_equal(a.counters, b.counters)


def test_single_pixel_stage_list_is_exact():
    # with only the pixel stage there is no level to approximate
    w = synth.scaled(3, 64, 64)
    p = synth.Params(w.params.n_superpixels, [1], 2, w.params.lambda_pos_q16)
    img = w.images()
    a = oracle.segment(img, p)
    p.stats_mode = synth.STATS_PYRAMID
    assert np.array_equal(a.labels, oracle.segment(img, p).labels)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_literal_mode_keeps_invariants(mode):
    # whatever the level data, the segmentation stays valid: every alive superpixel's pixel
    # count equals its label count, labels stay in range
    w = synth.scaled(3, 192, 192)
    p = synth.Params(w.params.n_superpixels, [16, 8, 4, 2, 1], 2, w.params.lambda_pos_q16, size_mode=mode,
                     stats_mode=synth.STATS_PYRAMID)
    o = oracle.segment(w.images(), p)
    counts = np.bincount(o.labels.ravel(), minlength=p.n_superpixels)
    assert np.array_equal(counts[o.sp["alive"] == 1], o.sp["n"][o.sp["alive"] == 1])

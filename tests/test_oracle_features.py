"""Pins of the f2 feature model of the oracle's prediction step (A31; Eq. 6): each
feature is isolated on a hand-built image whose value follows from the definition by hand,
and the Eq. 6 threshold (h = 0 -> y = +1) is probed one Q16 step either side of it."""
import copy

import numpy as np
import pytest

import oracle
import synth


def run(img, M, w):
    p = synth.Params(M, [2, 1], 1, synth.lambda_pos_default(img.shape[0], img.shape[1], M),
                     mask_rule=synth.MASK_CLASS, y_model=synth.Y_FEATURES, feat_w_q16=list(w))
    return oracle.segment(img[None], p).sp["y"]


def flat(v, H=8, W=8):
    return np.full((H, W, 3), v, np.uint8)


def test_f1_absolute_brightness_constant_image():
    # brightness 100 -> f1 = round(2^16 * 100 / 255) = 25700 (f2 = f3 = f4 = 0)
    f1 = (2 * 65536 * 100 + 255) // (2 * 255)
    assert f1 == 25700
    assert run(flat(100), 1, (-f1, 65536, 0, 0, 0)).tolist() == [1]      # h = 0 -> +1 (Eq. 6)
    assert run(flat(100), 1, (-f1 - 1, 65536, 0, 0, 0)).tolist() == [-1]
    # the f2 / f3 / f4 weights have no effect on a constant image with one superpixel
    assert run(flat(100), 1, (0, 0, -65536, -65536, -65536)).tolist() == [1]


def test_f3_intra_region_dissimilarity():
    # one superpixel, half the pixels brightness 0, half 200: variance 100^2 ->
    # f3 = round(2^16 * 100^2 / 255^2) = 10079
    img = flat(0)
    img[:, 4:] = 200
    f3 = (2 * 65536 * 100 ** 2 + 255 ** 2) // (2 * 255 ** 2)
    assert f3 == 10079
    assert run(img, 1, (-f3, 0, 0, 65536, 0)).tolist() == [1]
    assert run(img, 1, (-f3 - 1, 0, 0, 65536, 0)).tolist() == [-1]


def test_f2_comparative_and_f4_extra_region():
    # two superpixels (cells of 4 columns), brightness 100 | 200; image mean 150.  Q16 values
    # (round half up): f1 = 25700 | 51401, image 38551; f2 = -12851 | +12850;
    # f4 = |25700 - 51401| = 25701 for both
    img = flat(100)
    img[:, 4:] = 200
    rhu = lambda num, den: (2 * num + den) // (2 * den)  # noqa: E731
    f1a, f1b, f1i = rhu(65536 * 100, 255), rhu(65536 * 200, 255), rhu(65536 * 150, 255)
    assert (f1a, f1b, f1i) == (25700, 51401, 38551)
    assert run(img, 2, (12851, 0, 65536, 0, 0)).tolist() == [1, 1]       # left h = 0
    assert run(img, 2, (12850, 0, 65536, 0, 0)).tolist() == [-1, 1]
    assert run(img, 2, (-12850, 0, 65536, 0, 0)).tolist() == [-1, 1]     # right h = 0
    assert run(img, 2, (-12851, 0, 65536, 0, 0)).tolist() == [-1, -1]
    assert run(img, 2, (-25701, 0, 0, 0, 65536)).tolist() == [1, 1]      # f4 = 25701 for both
    assert run(img, 2, (-25702, 0, 0, 0, 65536)).tolist() == [-1, -1]


def test_weights_zero_and_negative_bias():
    # SPEC's classify examples: bias 0, theta 0 -> +1 (h = 0); bias -1 -> -1
    img = flat(100)
    img[:, 4:] = 200
    assert run(img, 2, (0, 0, 0, 0, 0)).tolist() == [1, 1]
    assert run(img, 2, (-65536, 0, 0, 0, 0)).tolist() == [-1, -1]


def test_feature_model_drives_the_mask():
    # tissue model (y = +1 iff mean brightness <= 0.85 * 255): on config 3's densities the
    # white background superpixels are inactive, and active == (y == +1) for alive ones
    w = synth.scaled(3, 256, 256)
    p = copy.deepcopy(w.params)
    p.y_model = synth.Y_FEATURES
    o = oracle.segment(w.images(), p)
    alive = o.sp["alive"] == 1
    assert np.array_equal(o.sp["active"][alive] == 1, o.sp["y"][alive] == 1)
    assert 0 < int((o.sp["y"][alive] == 1).sum()) < int(alive.sum())

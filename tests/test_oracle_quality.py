"""Pins of the f4 quality oracle (UE, BR, oracle.h) by hand-worked closed forms and
properties that hold for any input — not by re-implementing the definitions."""
import numpy as np
import pytest

import oracle


def halves(H, W, cut):
    g = np.zeros((H, W), np.int32)
    g[:, cut:] = 1
    return g


def test_identity_is_perfect():
    g = halves(8, 8, 4)
    q = oracle.quality(g, g, 0)
    assert q["ue"] == 0.0 and q["br"] == 1.0 and q["gt_boundary"] == 16  # columns 3 and 4


def test_single_superpixel_over_two_equal_segments():
    # each segment S contributes min(|S|, N - |S|) = N / 2: UE = 1 (SPEC's 4x4 example)
    g = halves(4, 4, 2)
    q = oracle.quality(np.zeros((4, 4), np.int32), g, 3)
    assert q["leak"] == 16 and q["ue"] == 1.0
    assert q["br"] == 0.0  # no superpixel boundary pixel exists


@pytest.mark.parametrize("k", [1, 2, 3, 5, 6])
def test_leak_of_k_pixels_counts_twice(k):
    # 6x6, GT halves at column 3; superpixel 0 = left half + k pixels of column 3:
    # S0 sees min(18, k) = k, S1 sees min(k, 18) = k -> UE = 2k / 36 (SPEC's 6x6 example)
    g = halves(6, 6, 3)
    lab = g.copy()
    lab.T.flat[18:18 + k] = 0  # the first k pixels of column 3
    assert int((lab[:, 3] == 0).sum()) == k
    q = oracle.quality(lab, g, 1)
    assert q["leak"] == 2 * k and q["ue"] == pytest.approx(2 * k / 36)


def test_displaced_cut_recall_by_eps():
    # GT edge between columns 3|4 (boundary columns 3, 4); cut one column right (boundary
    # columns 4, 5): column 4 coincides, column 3 is one pixel away
    g, lab = halves(8, 8, 4), halves(8, 8, 5)
    assert oracle.quality(lab, g, 0)["br"] == 0.5
    assert oracle.quality(lab, g, 1)["br"] == 1.0
    assert oracle.quality(lab, g, 2)["br"] == 1.0
    # two columns away: nothing at eps 0, column 4 only (one away) at eps 1, all at eps 2
    lab2 = halves(8, 8, 6)
    assert [oracle.quality(lab2, g, e)["br"] for e in (0, 1, 2)] == [0.0, 0.5, 1.0]


def test_no_gt_boundary_means_full_recall():
    q = oracle.quality(halves(5, 7, 3), np.full((5, 7), 9, np.int32), 0)
    assert q["gt_boundary"] == 0 and q["br"] == 1.0
    # one GT segment: every superpixel lies inside it -> no leak
    assert q["ue"] == 0.0


def test_properties_on_random_maps():
    rng = np.random.default_rng(5)
    for _ in range(20):
        H, W = rng.integers(3, 14, 2)
        g = rng.integers(0, 4, (H, W)).astype(np.int32)
        # a refinement of g (superpixels never straddle a segment): UE = 0, BR(0) = 1
        fine = (g * 1000 + rng.integers(0, 3, (H, W))).astype(np.int32)
        qf = oracle.quality(fine, g, 0)
        assert qf["ue"] == 0.0 and qf["br"] == 1.0
        lab = rng.integers(0, 5, (H, W)).astype(np.int32)
        brs = [oracle.quality(lab, g, e)["br"] for e in range(4)]
        assert all(0.0 <= b <= 1.0 for b in brs) and brs == sorted(brs)  # monotone in eps
        q = oracle.quality(lab, g, 1)
        assert 0.0 <= q["ue"] <= 1.0
        # a constant labelling: leak = sum_S min(|S|, N - |S|)
        qc = oracle.quality(np.zeros_like(g), g, 0)
        sizes = np.bincount(g.ravel())
        assert qc["leak"] == int(np.minimum(sizes, g.size - sizes)[sizes > 0].sum())


def test_batch_sums_images():
    g = np.stack([halves(6, 6, 3), halves(6, 6, 2)])
    lab = np.stack([halves(6, 6, 4), halves(6, 6, 2)])
    q = oracle.quality(lab, g, 0)
    q0, q1 = oracle.quality(lab[0], g[0], 0), oracle.quality(lab[1], g[1], 0)
    assert q["leak"] == q0["leak"] + q1["leak"] and q["covered"] == q0["covered"] + q1["covered"]
    assert q["gt_boundary"] == q0["gt_boundary"] + q1["gt_boundary"] and q["pixels"] == 72

"""Pins for O1 (grid), O2 (stage geometry), O3/O4 (block sums, S_1), O5 (rounding) and
the A9 topology test.  -m "not gpu"."""
from fractions import Fraction
import itertools

import numpy as np
import pytest

import oracle
import synth
import brute


# ---------------------------------------------------------------- O1
@pytest.mark.parametrize("H,W,M,expect", [
    (321, 481, 400, (16, 25)),     # config 1: 16x25 cells of 19-20 x 20-21 px
    (2048, 2048, 4096, (64, 64)),  # configs 2-5: square 32x32-px cells
    (8192, 8192, 65536, (256, 256)),
    (1024, 1024, 1024, (32, 32)),
    (8, 8, 2, (1, 2)),             # H1: tie -> fewer rows
    (4, 4, 4, (2, 2)),
    (4, 5, 4, (2, 2)),             # SPEC S:79 (5 wide x 4 tall)
    (7, 9, 1, (1, 1)),             # M=1: one label
])
def test_grid_known_values(H, W, M, expect):
    assert oracle.grid(H, W, M) == expect


def _brute_grid(H, W, M):
    best = None
    for r in range(1, M + 1):
        if M % r:
            continue
        c = M // r
        if c > W or r > H:
            continue
        a, b = W * r, H * c
        ratio = Fraction(max(a, b), min(a, b))
        if best is None or ratio < best[0]:
            best = (ratio, r, c)
    return best[1:]


def test_grid_brute_force_and_cells():
    rng = np.random.default_rng(0)
    for _ in range(300):
        H, W = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        M = int(rng.integers(1, min(H * W, 80) + 1))
        try:
            r, c = oracle.grid(H, W, M)
        except oracle.OracleError:
            assert all(not (M % r == 0 and M // r <= W and r <= H) for r in range(1, M + 1))
            continue
        assert (r, c) == _brute_grid(H, W, M)
        X = [(i * W) // c for i in range(c + 1)]
        Y = [(j * H) // r for j in range(r + 1)]
        assert min(np.diff(X)) >= 1 and min(np.diff(Y)) >= 1  # no empty cell
        assert max(np.diff(X)) - min(np.diff(X)) <= 1          # areas differ by <= 1 row/col


# ---------------------------------------------------------------- O2
def test_config1_stage_block_counts():
    w = synth.config(1)
    geo = brute.geometry(w.H, w.W, w.params.n_superpixels, w.params.block_sizes)
    counts = [(len(xs) - 1, len(ys) - 1) for xs, ys in geo]
    # 51x33, 81x49, 139x81, 253x161 and 481x321 blocks
    assert counts == [(51, 33), (81, 49), (139, 81), (253, 161), (481, 321)]
    assert [a * b for a, b in counts[:4]] == [1683, 3969, 11259, 40733]


def test_stage_axes_nested_and_cells_respected():
    rng = np.random.default_rng(1)
    for _ in range(100):
        H, W = int(rng.integers(8, 90)), int(rng.integers(8, 90))
        M = int(rng.integers(1, 30))
        try:
            r, c = oracle.grid(H, W, M)
        except oracle.OracleError:
            continue
        sizes = [16, 8, 4, 2, 1]
        geo = brute.geometry(H, W, M, sizes)
        X = [(i * W) // c for i in range(c + 1)]
        for s, (xs, ys) in enumerate(geo):
            assert xs[0] == 0 and xs[-1] == W and np.all(np.diff(xs) >= 1)
            assert set(X) <= set(xs.tolist())              # blocks never straddle a cell
            assert np.all(np.diff(xs) <= sizes[s])          # block widths <= b_s
            if s + 1 < len(geo):
                assert set(xs.tolist()) <= set(geo[s + 1][0].tolist())  # xs_s subset of xs_{s+1}
        assert list(geo[-1][0]) == list(range(W + 1))       # pixel stage


# ---------------------------------------------------------------- O5 (A24)
def test_round_mean_exhaustive():
    for n in range(1, 41):
        for S in range(0, 255 * n + 1, max(1, n // 3)):
            want = brute.round_half_up(Fraction(S * 256, n))
            assert oracle.round_mean(S, n) == want, (S, n)
    # large sums (position sums of a 1-Gpx image)
    for S, n in [(2**45 + 12345, 2**30 - 7), (2**40, 3), (10**12 + 1, 2)]:
        assert oracle.round_mean(S, n) == brute.round_half_up(Fraction(S * 256, n))


# ---------------------------------------------------------------- O5 + A33 (colour means)
def test_colour_mean_clamped_to_intensity_range():
    # inside [0, 255 n] the colour mean is O5's rounding; a constant region of intensity v has
    # mean v exactly (v * 2^8); outside the range (literal pyramid data only) the mean is the
    # nearest intensity bound, 0 or 255 (DESIGN A33)
    for n in range(1, 25):
        for v in (0, 1, 128, 254, 255):
            assert oracle.colour_mean(v * n, n) == v << 8
        for S in range(-3 * n, 258 * n, max(1, n // 2)):
            exact = brute.round_half_up(Fraction(S * 256, n))
            want = 0 if S < 0 else (255 << 8 if S > 255 * n else exact)
            assert oracle.colour_mean(S, n) == want, (S, n)
            if 0 <= S <= 255 * n:
                assert oracle.colour_mean(S, n) == oracle.round_mean(S, n)
    assert oracle.colour_mean(-1, 10**6) == 0                 # rounds to 0 anyway
    assert oracle.colour_mean(255 * 7 + 1, 7) == 255 << 8      # just above the range
    assert oracle.colour_mean(-(2**40), 3) == 0


# ---------------------------------------------------------------- A9 (E_topo)
def test_topology_lut_exhaustive_vs_flood_fill():
    accepted = 0
    reachable = 0
    for m in range(256):
        edge = sum((m >> k) & 1 for k in (0, 2, 4, 6))
        if not (1 <= edge <= 3):
            continue
        reachable += 1
        simple = brute.local_simple(m)
        assert (oracle.yokoi_c4(m) == 1) == simple, m
        accepted += simple
    assert reachable == 224 and accepted == 112
    assert oracle.yokoi_c4(0) == 0      # isolated / last block of A
    assert oracle.yokoi_c4(0b00010001) == 2  # 1-wide vertical bridge N-S: two runs
    assert oracle.yokoi_c4(0b00011100) == 1  # convex corner of a solid 2x2


# ---------------------------------------------------------------- O3/O4
@pytest.mark.parametrize("k", [1, 5])
def test_stage_sums_equal_recount(k):
    """At every stage start the reused sums (S_1 from pixels, moved block sums) equal a
    recount from the pixel-expanded map (A23: Eq. 8 is exact at full resolution)."""
    w = synth.config(k) if k == 1 else synth.scaled(5, 128, 96, B=2)
    img = w.images()
    p = w.params
    geo = brute.geometry(w.H, w.W, p.n_superpixels, p.block_sizes)
    for s in range(len(p.block_sizes)):
        res = oracle.segment(img, p, stop=(oracle.STOP_STAGE_START, s, 0, 0))
        for b in range(w.B):
            pix = brute.expand(res.map[b], *geo[s])
            M = p.n_superpixels
            want = brute.recount(img[b], pix, M)
            got = brute.sp_sums(res.sp[b * M:(b + 1) * M])
            assert np.array_equal(got, want)
            if s == 0:  # initial grid: InitSize = cell area = n
                assert np.array_equal(res.sp["init_size"][b * M:(b + 1) * M], want[:, 0])

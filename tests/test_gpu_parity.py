"""GPU parity: the sm_100a path (called through the C ABI) against the CPU oracle, element
by element, on seeded synthetic inputs.  Bar: bit-exact labels, exact int64 sums, identical
flags and per-phase move counts; derived float means within 1e-6 relative."""
import copy

import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_parity, gpu_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rapid():
    import torch
    import paper_1704_02083_b200 as rb
    assert torch.cuda.is_available()
    r = rb.Rapid(0, max_pixels=1 << 27, max_superpixels=1 << 17)
    yield r
    r.close()


def P(M, sizes, sweeps=3, lam_pos=65536, lam_b=32 * 65536, size_mode=0, mask=0, l=(1, 4),
      u=(3, 2), tau2=1600, stats=0):
    return synth.Params(M, list(sizes), sweeps, lam_pos, lam_b, size_mode, l[0], l[1], u[0], u[1],
                        mask, [synth.PROTO_PINK, synth.PROTO_PURPLE], tau2, stats)


# ----------------------------------------------------------------------- hand-worked H1
def test_H1_on_gpu(rapid):
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    img[:, 3:, :] = 200
    o, lab, sp, info = assert_parity(rapid, img, P(2, [2, 1], 2))
    want = np.zeros((8, 8), dtype=np.int32)
    want[:, 3:] = 1
    assert np.array_equal(lab[0], want)
    assert info.counters()[1, 0, :, oracle.C_COMMIT].tolist() == [0, 4, 0, 4]


# ----------------------------------------------------------------------- full configs
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_config1_full(rapid, mode):
    w = synth.config(1)
    p = copy.deepcopy(w.params)
    p.size_mode = mode
    assert_parity(rapid, w.images(), p)


def test_config1_recount_equals_reuse(rapid):
    w = synth.config(1)
    p = copy.deepcopy(w.params)
    p.stats_mode = synth.STATS_RECOUNT
    o, lab, sp, info = assert_parity(rapid, w.images(), p)
    assert info.status == 0


def test_config2_full(rapid):
    w = synth.config(2)
    assert_parity(rapid, w.images(), w.params)


@pytest.mark.slow
def test_config3_full(rapid):
    w = synth.config(3)
    o, lab, sp, info = assert_parity(rapid, w.images(), w.params)
    assert 0 < info.active < info.alive


@pytest.mark.slow
def test_config5_batch_full(rapid):
    w = synth.config(5)
    assert_parity(rapid, w.images(), w.params)


def test_config4_scaled_sample(rapid):
    """config 4's densities, prediction mask and merges at 2048^2 (full pipeline)."""
    w = synth.scaled(4, 2048, 2048)
    assert_parity(rapid, w.images(), w.params)


# ----------------------------------------------------------------------- random cases
def _cases(seed, n):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        H, W = int(rng.integers(17, 150)), int(rng.integers(17, 150))
        M = int(rng.integers(2, max(3, H * W // 150)))
        try:
            oracle.grid(H, W, M)
        except oracle.OracleError:
            continue
        regions = int(rng.integers(2, 12))
        img = synth.image(H, W, int(rng.integers(1 << 30)), regions, int(rng.integers(0, 30)),
                          int(rng.integers(0, 400)))
        sizes = [[8, 4, 2, 1], [16, 8, 4, 2, 1], [4, 2, 1], [4, 1], [2], [8, 4], [32, 16, 8, 4, 2, 1]][
            int(rng.integers(7))]
        yield rng, img, M, sizes


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_random_small_all_size_modes(rapid, mode):
    for rng, img, M, sizes in _cases(100 + mode, 12):
        p = P(M, sizes, int(rng.integers(1, 5)), int(rng.integers(0, 6 * 65536)),
              int(rng.integers(0, 64 * 65536)), size_mode=mode)
        assert_parity(rapid, img, p)


@pytest.mark.parametrize("mask", [1, 2, 3])
def test_random_small_mask_rules(rapid, mask):
    for rng, img, M, sizes in _cases(200 + mask, 10):
        p = P(M, sizes, 3, size_mode=int(rng.integers(0, 3)), mask=mask,
              tau2=int(rng.integers(200, 6000)))
        assert_parity(rapid, img, p)


def test_random_batches(rapid):
    rng = np.random.default_rng(7)
    for _ in range(4):
        B = int(rng.integers(2, 6))
        H, W = int(rng.integers(40, 120)), int(rng.integers(40, 120))
        imgs = np.stack([synth.image(H, W, int(rng.integers(1 << 30)), 6, 20, 200) for _ in range(B)])
        p = P(12, [8, 4, 2, 1], 3, size_mode=2, mask=int(rng.integers(0, 4)))
        o, lab, sp, info = assert_parity(rapid, imgs, p)
        for b in range(B):  # batch == singles
            l1, sp1, _ = gpu_run(rapid, imgs[b], p)
            assert np.array_equal(l1[0], lab[b])


# ----------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("H,W,M,sizes", [
    (1, 1, 1, [1]),
    (1, 40, 4, [4, 2, 1]),
    (37, 1, 3, [2, 1]),
    (5, 7, 35, [4, 2, 1]),        # every pixel its own superpixel
    (64, 64, 1, [32, 16, 1]),     # M = 1: nothing moves
    (130, 70, 9, [64, 32, 16, 8, 4, 2, 1]),  # maximum block size
    (33, 65, 6, [8, 4]),          # final grain 4 with ragged borders
])
def test_edge_shapes(rapid, H, W, M, sizes):
    img = synth.image(H, W, 11, 3, 2, 0)
    for mode in (0, 2):
        assert_parity(rapid, img, P(M, sizes, 3, size_mode=mode))


def test_zero_sweeps_and_constant_image(rapid):
    img = synth.image(96, 80, 5, 5, 10, 0)
    assert_parity(rapid, img, P(20, [8, 4, 2, 1], 0))
    const = np.full((64, 96, 3), 77, dtype=np.uint8)
    o, lab, sp, info = assert_parity(rapid, const, P(24, [8, 4, 2, 1], 3, size_mode=2))
    assert info.counters()[..., oracle.C_COMMIT].sum() == 0


def test_determinism_and_host_api(rapid):
    w = synth.config(2)
    img = w.images()
    l1, s1, _ = gpu_run(rapid, img, w.params)
    l2, s2, _ = gpu_run(rapid, img, w.params)
    assert np.array_equal(l1, l2) and np.array_equal(s1, s2)
    lh = rapid.segment_host(img, w.params)
    assert np.array_equal(lh, l1)


def test_debug_stop_points_match_oracle(rapid):
    import torch
    w = synth.config(1)
    img = w.images()
    p = copy.deepcopy(w.params)
    p.size_mode = 2
    t = torch.from_numpy(img).cuda()
    cap = (w.H + 2) * (w.W + 2) * 2
    for pt in [(oracle.STOP_STAGE_START, 2, 0, 0), (oracle.STOP_PHASE, 3, 1, 2),
               (oracle.STOP_AFTER_MERGE, 3, 0, 0), (oracle.STOP_PHASE, 4, 0, 3)]:
        o = oracle.segment(img, p, stop=pt, map_cap=cap)
        rapid.debug_stop(*pt)
        rapid.segment(t, p)
        torch.cuda.synchronize()
        g = rapid.debug_map(cap)
        rapid.debug_stop(0)
        assert np.array_equal(g, o.map), pt


# ----------------------------------------------------------------------- randomized sweep
def test_random_all_options_combined(rapid):
    """Random small cases over every option at once (size mode, mask rule, y model, stats
    mode, lambdas, stage lists, final grain, batches), each bit-exact with the oracle."""
    import os
    random_all_options(rapid, int(os.environ.get("RAPID_RANDOM_SEED", "2024")),
                       int(os.environ.get("RAPID_RANDOM_CASES", "24")))


def random_all_options(rapid, seed, n):
    rng = np.random.default_rng(seed)
    for case in range(n):
        B = int(rng.integers(1, 4))
        H, W = int(rng.integers(24, 140)), int(rng.integers(24, 140))
        imgs = np.stack([synth.image(H, W, int(rng.integers(1 << 30)), int(rng.integers(2, 12)),
                                     int(rng.integers(0, 40)), int(rng.integers(0, 600))) for _ in range(B)])
        while True:  # a superpixel count whose grid fits the image
            M = int(rng.integers(1, max(2, H * W // 60)))
            try:
                oracle.grid(H, W, M)
                break
            except oracle.OracleError:
                pass
        top = int(rng.choice([8, 16, 32]))
        sizes = [top >> k for k in range(int(np.log2(top)) + 1)]
        if rng.random() < 0.3:
            sizes = sizes[:-2]  # final grain 4
        mask = int(rng.integers(0, 4))
        p = P(M, sizes, int(rng.integers(1, 5)), int(rng.integers(0, 4 * 65536)), int(rng.integers(0, 64 * 65536)),
              size_mode=int(rng.integers(0, 3)), mask=mask, tau2=int(rng.integers(200, 6000)),
              stats=int(rng.choice([0, 1, 2])))
        if mask and rng.random() < 0.5:
            p.y_model = synth.Y_FEATURES
            p.feat_w_q16 = [int(v) for v in rng.integers(-70000, 70000, 5)]
        try:
            assert_parity(rapid, imgs, p)
        except AssertionError as e:
            raise AssertionError(f"case {case}: B={B} H={H} W={W} params={p}: {e}") from None


# ----------------------------------------------------------------------- hand-worked H2-H4, ties
# (expected outputs worked out by hand in tests/test_oracle_choice.py; here the CUDA path must
#  give the same maps, sums and counters as the oracle and the hand-worked result)
def test_eq3_exact_ties_on_gpu(rapid):
    from test_oracle_choice import _two_by_two
    for colours, corner, want in [((100, 200, 200, 200), (3, 3), 1), ((200, 100, 200, 200), (4, 3), 0)]:
        img = _two_by_two(colours, corner, 200)
        o, lab, sp, info = assert_parity(rapid, img, P(4, [1], 1, lam_pos=0, lam_b=32 * 65536))
        exp = np.repeat(np.repeat(np.array([[0, 1], [2, 3]], np.int32), 4, 0), 4, 1)
        exp[corner[1], corner[0]] = want
        assert np.array_equal(lab[0], exp)


def test_H2_bridge_on_gpu(rapid):
    from test_oracle_choice import _h2_image
    o, lab, sp, info = assert_parity(rapid, _h2_image(), P(2, [1], 2, lam_pos=65536, lam_b=32 * 65536))
    want = np.ones((6, 6), dtype=np.int32)
    want[0, 0:3] = want[5, 0:3] = 0
    want[1:5, 0] = 0
    assert np.array_equal(lab[0], want)


@pytest.mark.parametrize("mode,u,mid,T", [(0, (3, 2), 200, None), (1, (3, 2), 200, None), (2, (3, 2), 200, None),
                                         (2, (7, 4), 200, 0), (2, (7, 4), 150, 2)])
def test_H3_size_modes_on_gpu(rapid, mode, u, mid, T):
    from test_oracle_choice import _h3_image, H3_HARD
    p = P(3, [2], 2, lam_pos=0, lam_b=65536, size_mode=mode, l=(1, 2), u=u)
    o, lab, sp, info = assert_parity(rapid, _h3_image(mid), p)
    if mode == 0:
        want = np.array([[0, 0, 0, 2, 2, 2], [0, 0, 0, 1, 2, 2]], np.int32)
    else:
        want = H3_HARD if T is None else np.where(H3_HARD == 1, T, H3_HARD)
    assert np.array_equal(lab[0][::2, ::2], want)
    assert list(info.stage_merges)[0] == (0 if T is None else 1)


@pytest.mark.parametrize("rule", [1, 2, 3])
def test_H4_gating_on_gpu(rapid, rule):
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    img[:, 3:, :] = 200
    p = P(2, [2, 1], 2, mask=rule, tau2=100)
    p.protos = [(200, 200, 200)]
    o, lab, sp, info = assert_parity(rapid, img, p)
    want = np.zeros((8, 8), dtype=np.int32)
    want[:, 4 if rule == 1 else 3:] = 1
    assert np.array_equal(lab[0], want)
    assert sp["y"].tolist() == [-1, 1]


# ----------------------------------------------------------------------- 64-bit K4 variant
def test_config4_strip_reaches_64bit_block_stage(rapid):
    """A 128 x 32768 strip with config 4's densities, prediction and merges: at the b = 16 stage
    (max block area) x (max coordinate) = 256 x 32767 >= 2^22, so K4 runs its 64-bit
    position-factor variant (as config 4 itself does at b = 16) with real moves; labels, int64
    sums, flags and per-phase counters bit-exact with the oracle."""
    w = synth.scaled(4, 128, 32768)
    assert 16 * 16 * (32768 - 1) >= 1 << 22
    o, lab, sp, info = assert_parity(rapid, w.images(), w.params)
    s16 = w.params.block_sizes.index(16)
    assert o.counters[s16, ..., oracle.C_COMMIT].sum() > 100  # the 64-bit stage really moves blocks


def test_maximum_sweeps_and_stages(rapid):
    """The largest sweep count the ABI accepts (64, most of them skipped by the exact early exit)
    and a 7-stage list up to the largest block size, under MERGE with a mask: bit-exact, and the
    per-phase counters of every executed sweep equal the oracle's."""
    img = synth.image(144, 208, 77, 9, 60, 300)
    p = P(24, [64, 32, 16, 8, 4, 2, 1], 64, size_mode=2, mask=1, tau2=3000)
    o, lab, sp, info = assert_parity(rapid, img, p)
    assert max(int(x) for x in info.stage_sweeps_run[:7]) < 64  # the early exit did stop stages


@pytest.mark.parametrize("mask,stats,size_mode", [(2, 0, 2), (3, 0, 2), (1, 1, 2), (1, 2, 2), (1, 0, 1), (0, 1, 1)])
def test_config4_density_options_at_2048(rapid, mask, stats, size_mode):
    """Config 4's densities at 2048^2 (4096 superpixels, 2048 worklist-sized tiles at the pixel
    stage) under the other mask rules (BSP, EQ7), stats modes (RECOUNT, PYRAMID) and size modes
    (HARD with and without the mask): bit-exact with the oracle, counters included."""
    w = synth.scaled(4, 2048, 2048)
    p = copy.deepcopy(w.params)
    p.mask_rule, p.stats_mode, p.size_mode = mask, stats, size_mode
    o, lab, sp, info = assert_parity(rapid, w.images(), p)
    assert info.status == 0


def test_random_midsize_config4_densities(rapid):
    """Random mid-size cases with config 4's densities (ragged sizes of several 32 x 32 tiles
    up to ~1.5 Mpx, so that worklists, multi-tile boundary sets, merges and the prediction mask
    all engage), random options, each bit-exact with the oracle.  RAPID_MIDSIZE_SEED /
    RAPID_MIDSIZE_CASES widen the sweep (profiles/r02j_soak.txt)."""
    import os
    rng = np.random.default_rng(int(os.environ.get("RAPID_MIDSIZE_SEED", "77")))
    for case in range(int(os.environ.get("RAPID_MIDSIZE_CASES", "6"))):
        H, W = int(rng.integers(200, 1300)), int(rng.integers(200, 1300))
        w = synth.scaled(4, H, W, B=int(rng.integers(1, 3)), seed_offset=int(rng.integers(1 << 20)))
        p = w.params
        while True:  # a superpixel count whose grid fits the image (A1: M = rows x columns)
            try:
                oracle.grid(H, W, p.n_superpixels)
                break
            except oracle.OracleError:
                p.n_superpixels -= 1
        p.sweeps = int(rng.integers(1, 6))
        p.size_mode = int(rng.integers(0, 3))
        p.mask_rule = int(rng.integers(0, 4))
        p.stats_mode = int(rng.choice([0, 0, 1, 2]))
        p.lambda_b_q16 = int(rng.integers(0, 64 * 65536))
        if rng.random() < 0.3:
            p.block_sizes = p.block_sizes[:-int(rng.integers(1, 3))]  # final grain 2 or 4
        try:
            assert_parity(rapid, w.images(), p)
        except AssertionError as e:
            raise AssertionError(f"case {case}: {w.name} B={w.B} params={p}: {e}") from None

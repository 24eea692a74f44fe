"""Pins for the oracle's CHOICES (-m "not gpu"): which move Eq. 3 picks (argmin over
the 4-neighbour labels, A7: ties to the lowest id, move only if dE < 0) and which target Eq. 4
picks (argmin over the contiguous superpixels that pass Eq. 5, A19: victims in
ascending id, locks; A13-A16).  The expected choices are recomputed here by brute force from
the paper's definitions (tests/brute.py: per-pixel Eq. 1 + Eq. 2 energy, flood-fill simple
points); nothing here calls the oracle's energy, topology or argmin code.  Plus the hand-worked
cases H2 (bridge), H3 (size modes) and H4 (gating) of SURVEY §8(c) and two constructed exact
ties, with expected outputs worked out by hand in the comments."""
import copy

import numpy as np
import pytest

import oracle
import synth
import brute
from test_oracle_energy import params, cut_image, before_key, state, dE_of

RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]  # N NE E SE S SW W NW
N4 = [(0, -1), (1, 0), (0, 1), (-1, 0)]


def ring_mask(bmap, i, j):
    H, W = bmap.shape
    A = bmap[j, i]
    m = 0
    for k, (dx, dy) in enumerate(RING):
        x, y = i + dx, j + dy
        if 0 <= x < W and 0 <= y < H and bmap[y, x] == A:
            m |= 1 << k
    return m


def brute_phase(img, bmap, sums, xs, ys, ph, lp, lb):
    """Expected result of one phase (size NONE, mask OFF) by brute force: for every block of
    the phase colour that is a boundary block and a simple point (flood-fill definition), the
    energy change of relabelling it to each distinct 4-neighbour label B != A (full per-pixel
    recomputation under the frozen snapshot means); B* = argmin (dE, B); moves iff dE(B*) < 0.
    Returns (expected map, #ties at the minimum, #moves, #blocks evaluated)."""
    H, W = bmap.shape
    cq, mq = brute.quantised_means(sums)
    E0 = brute.energy_int(img, brute.expand(bmap, xs, ys), cq, mq, lp, lb)
    out = bmap.copy()
    ties = moves = evaluated = 0
    for j in range(ph >> 1, H, 2):
        for i in range(ph & 1, W, 2):
            A = bmap[j, i]
            nb = [bmap[j + dy, i + dx] for dx, dy in N4 if 0 <= i + dx < W and 0 <= j + dy < H]
            if all(q == A for q in nb):
                continue
            if not brute.local_simple(ring_mask(bmap, i, j)):
                continue
            scores = []
            evaluated += 1
            for B in sorted(set(int(q) for q in nb) - {int(A)}):
                one = bmap.copy()
                one[j, i] = B
                scores.append((brute.energy_int(img, brute.expand(one, xs, ys), cq, mq, lp, lb) - E0, B))
            best = min(scores)
            ties += sum(1 for s in scores if s[0] == best[0]) > 1
            if best[0] < 0:
                out[j, i] = best[1]
                moves += 1
    return out, ties, moves, evaluated


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        H, W = int(rng.integers(8, 15)), int(rng.integers(8, 15))
        M = int(rng.integers(2, 9))
        try:
            oracle.grid(H, W, M)
        except oracle.OracleError:
            continue
        img = cut_image(rng, H, W) if rng.random() < 0.6 else rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        sizes = [[2, 1], [4, 2, 1], [1]][int(rng.integers(3))]
        yield img, H, W, M, sizes, int(rng.integers(0, 4 * 65536)), int(rng.integers(0, 48 * 65536))


def test_eq3_choice_is_brute_force_argmin_every_phase():
    """Every block of every phase of random runs: the oracle's new label is the brute-force
    argmin of Eq. 1 over the distinct 4-neighbour labels (lowest id on ties), only when that
    minimum is < 0, and only for simple boundary blocks; every other block keeps its label."""
    decisions = moves = 0
    for img, H, W, M, sizes, lp, lb in _cases(12, 31):
        p = params(M, sizes, 2, lp, lb)
        geo = brute.geometry(H, W, M, sizes)
        for s in range(len(sizes)):
            xs, ys = geo[s]
            for t in range(p.sweeps):
                for ph in range(4):
                    bmap, bsums, _ = state(img, p, before_key(p, s, t, ph))
                    amap, _, _ = state(img, p, (oracle.STOP_PHASE, s, t, ph))
                    want, _, mv, ev = brute_phase(img, bmap, bsums, xs, ys, ph, lp, lb)
                    assert np.array_equal(amap, want), (s, t, ph, np.argwhere(amap != want)[:4].tolist())
                    decisions += ev
                    moves += mv
    assert decisions > 1000 and moves > 150 and decisions > moves


def _two_by_two(colour_of_cell, corner, corner_colour):
    """8x8 image, M = 4 -> 2x2 grid of 4x4 cells (labels 0 1 / 2 3), flat colours, one
    corner pixel recoloured."""
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    for lab, c in enumerate(colour_of_cell):
        y0, x0 = 4 * (lab // 2), 4 * (lab % 2)
        img[y0:y0 + 4, x0:x0 + 4] = c
    x, y = corner
    img[y, x] = corner_colour
    return img


@pytest.mark.parametrize("lam_b", [1, 32])
def test_eq3_exact_tie_goes_to_lowest_label(lam_b):
    """A7 tie, worked by hand.  Case 1: cells 0 = 100, 1 = 2 = 3 = 200, pixel (3,3) of cell 0
    = 200.  Its E neighbour is label 1 and its S neighbour label 2, both with quantised mean
    exactly 200 (F = 8), lambda_pos = 0; dB2 is +2 for either (N, W stay label 0), so dE(1) ==
    dE(2) < 0 (dC = -3 (200 - c_0)^2 with c_0 = 106.25): the pixel must go to label 1.
    Ring N NE E SE S SW W NW = 0 1 1 3 2 2 0 0 -> C4 = 1 (simple).
    Case 2 (the lower id later in N, E, S, W scan order): cells 1 = 100, 0 = 2 = 3 = 200, pixel
    (4,3) of cell 1 = 200: S neighbour label 3, W neighbour label 0, dB2 = +2 for both ->
    label 0.  Every other pixel keeps its label (a move between the 200 cells has dC = 0 and
    dB2 >= 0; a 100-pixel gains nothing from a 200 mean).  Stages [1], 1 sweep, NONE."""
    for colours, corner, want in [((100, 200, 200, 200), (3, 3), 1), ((200, 100, 200, 200), (4, 3), 0)]:
        img = _two_by_two(colours, corner, 200)
        p = params(4, [1], 1, 0, lam_b * 65536)
        r = oracle.segment(img, p, log_moves=10)
        exp = np.repeat(np.repeat(np.array([[0, 1], [2, 3]], np.int32), 4, 0), 4, 1)
        exp[corner[1], corner[0]] = want
        assert np.array_equal(r.labels[0], exp), r.labels[0]
        assert len(r.moves) == 1 and int(r.moves[0]["B"]) == want
        # the two candidates really tie (brute force), and the move is a descent
        x, y = corner
        A = int(np.repeat(np.repeat(np.array([[0, 1], [2, 3]]), 4, 0), 4, 1)[y, x])
        bmap = np.repeat(np.repeat(np.array([[0, 1], [2, 3]], np.int32), 4, 0), 4, 1)
        sums = brute.recount(img, bmap, 4)
        cq, mq = brute.quantised_means(sums)
        E0 = brute.energy_int(img, bmap, cq, mq, 0, lam_b * 65536)
        dE = {}
        for B in {int(bmap[y, x + 1]), int(bmap[y + 1, x]), int(bmap[y, x - 1]), int(bmap[y - 1, x])} - {A}:
            one = bmap.copy()
            one[y, x] = B
            dE[B] = brute.energy_int(img, one, cq, mq, 0, lam_b * 65536) - E0
        cands = sorted(dE)
        assert len(cands) == 2 and dE[cands[0]] == dE[cands[1]] < 0 and want == cands[0]


def _h2_image():
    img = np.full((6, 6, 3), 200, dtype=np.uint8)
    img[0, 0:3] = 0
    img[5, 0:3] = 0
    return img


@pytest.mark.parametrize("lam_pos,lam_b", [(0, 0), (0, 1), (1, 32), (10, 100)])
def test_H2_bridge_never_moves(lam_pos, lam_b):
    """H2, worked by hand.  6x6, M = 2 -> labels A = 0 (x < 3), B = 1 (x >= 3).  A's rows 0
    and 5 are dark (0), everything else 200, so every 200 pixel of A prefers B (dC_real per
    channel -(200 - c_A)^2, c_A in [80, 133]) by far more than any boundary / position change.
    Sweep 0 (pixel stage only) erodes A's 200 pixels from the right: phase (0,0) moves (2,2),
    (2,4); (1,0) moves (1,2), (1,4); (0,1) moves (2,1), (2,3); (1,1) moves (1,1), (1,3).  What
    is left of A is the two dark rows joined by the 1-pixel-wide bridge x = 0, y = 1..4.  Every
    bridge pixel has C4 = 2 (e.g. (0,2): ring N NE E SE S SW W NW = A B B B A - - -), so it
    never moves although its colour favours B: A stays 4-connected.  Sweep 1 makes no move."""
    img = _h2_image()
    p = params(2, [1], 2, lam_pos * 65536, lam_b * 65536)
    r = oracle.segment(img, p, log_moves=100)
    want = np.ones((6, 6), dtype=np.int32)
    want[0, 0:3] = 0
    want[5, 0:3] = 0
    want[1:5, 0] = 0
    assert np.array_equal(r.labels[0], want), r.labels[0]
    c = r.counters[0, :2, :, oracle.C_COMMIT]
    assert c.tolist() == [[2, 2, 2, 2], [0, 0, 0, 0]]
    # sweep 1: the bridge pixels of the phase colours (0,0) and (0,1) are candidates whose
    # topology test fails; had they been allowed to move, the energy would have dropped
    assert r.counters[0, 1, 0, oracle.C_CAND] > r.counters[0, 1, 0, oracle.C_TOPO]
    sums = brute.recount(img, want, 2)
    cq, mq = brute.quantised_means(sums)
    E0 = brute.energy_int(img, want, cq, mq, lam_pos * 65536, lam_b * 65536)
    for y in range(1, 5):
        one = want.copy()
        one[y, 0] = 1
        assert brute.energy_int(img, one, cq, mq, lam_pos * 65536, lam_b * 65536) < E0
        assert not brute.local_simple(ring_mask(want, 0, y))
    assert brute.all_connected(r.labels[0])


def _h3_image(mid_left=200):
    """4x12, M = 3 -> 1x3 grid of 4x4 cells; stage b = 2 gives a 6x2 block grid, labels
    0 = block columns 0-1, 1 = 2-3, 2 = 4-5.  Cell 0 = 200, cell 2 = 0; the middle cell's block
    column 2 is like its left neighbour (200, or `mid_left` in its lower block) and block
    column 3 like its right neighbour (0)."""
    img = np.zeros((4, 12, 3), dtype=np.uint8)
    img[:, 0:8] = 200
    img[2:4, 4:6] = mid_left
    img[:, 6:8] = 0
    return img


H3_HARD = np.array([[0, 0, 0, 2, 2, 2], [0, 0, 1, 1, 2, 2]], np.int32)


@pytest.mark.parametrize("lam_b", [0, 1, 32])
def test_H3_size_modes(lam_b):
    """H3, worked by hand (stage b = 2 only, lambda_pos = 0, l = 1/2 -> floor 8 px = 2 blocks).
    Sweep 0: (0,0) moves block (2,0) to 0 (dC = -4*3*100^2, c_1 = 100); (1,0) moves (3,0) to 2
    (c_1 = 66.7 -> 0 is closer than 200); (0,1) wants (2,1) -> 0 and (1,1) wants (3,1) -> 2
    (C4 = 1 with (2,1) still in the middle superpixel).
      NONE: both commit ((3,1) has C4 = 0 after (2,1) left, so it stays): the middle
            superpixel ends with one block, 4 px < the floor.  Nothing moves in sweep 1
            (lambda_pos = 0: equal colour means give dE = 0, not < 0).
      HARD: (2,1) and (3,1) are size-rejected ((8 - 4)*2 < 16): the middle keeps exactly the
            floor, 8 px; the same two rejections repeat in sweep 1.
      MERGE, u = 3/2: it is a victim, but both neighbours would exceed u: (20 + 8)*2 > 3*16
            (Eq. 5) -> no merge (A16), same map as HARD.
      MERGE, u = 7/4: both bounds hold, dE_m(1->0) == dE_m(1->2) (dC = 3*80000 for either,
            -2*len*lambda_b with len = 4 for either): exact tie -> the lower id, T = 0.
      MERGE, u = 7/4 with the middle's lower-left block at 150: dE_m(1->0) = 3*125000 >
            dE_m(1->2) = 3*45000 -> T = 2."""
    img = _h3_image()
    base = params(3, [2], 2, 0, lam_b * 65536, l=(1, 2), u=(3, 2))
    none = copy.deepcopy(base); none.size_mode = synth.SIZE_NONE
    r = oracle.segment(img, none)
    want_none = np.array([[0, 0, 0, 2, 2, 2], [0, 0, 0, 1, 2, 2]], np.int32)
    assert np.array_equal(r.labels[0][::2, ::2], want_none)
    assert r.sp["n"].tolist() == [24, 4, 20]
    assert r.counters[0, :2, :, oracle.C_COMMIT].tolist() == [[1, 1, 1, 0], [0, 0, 0, 0]]

    hard = copy.deepcopy(base); hard.size_mode = synth.SIZE_HARD
    r = oracle.segment(img, hard)
    assert np.array_equal(r.labels[0][::2, ::2], H3_HARD)
    assert r.sp["n"].tolist() == [20, 8, 20]
    assert r.counters[0, :2, :, oracle.C_COMMIT].tolist() == [[1, 1, 0, 0], [0, 0, 0, 0]]
    assert r.counters[0, :2, :, oracle.C_SIZEREJ].tolist() == [[0, 0, 1, 1], [0, 0, 1, 1]]

    merge = copy.deepcopy(base); merge.size_mode = synth.SIZE_MERGE
    r = oracle.segment(img, merge, log_merges=4)
    assert np.array_equal(r.labels[0][::2, ::2], H3_HARD) and len(r.merges) == 0
    assert r.stage_victims[0] == 1 and r.stage_merges[0] == 0

    for mid, T in [(200, 0), (150, 2)]:
        m2 = copy.deepcopy(merge); m2.u_num, m2.u_den = 7, 4
        r = oracle.segment(_h3_image(mid), m2, log_merges=4)
        assert len(r.merges) == 1 and (int(r.merges[0]["A"]), int(r.merges[0]["T"])) == (1, T)
        want = np.where(H3_HARD == 1, T, H3_HARD)
        assert np.array_equal(r.labels[0][::2, ::2], want)
        assert r.sp["alive"].tolist() == [1, 0, 1] and r.sp["n"][T] == 28
        assert int(r.merges[0]["len"]) == 4


def _h1_image():
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    img[:, 3:, :] = 200
    return img


@pytest.mark.parametrize("rule", [1, 2, 3])
def test_H4_gating(rule):
    """H4, worked by hand: H1's image (columns 0-2 = 0, 3-7 = 200; labels 0 = x < 4, 1 =
    x >= 4; stages [2, 1]) with the prototype (200,200,200) and tau^2 = 100.  Prediction after
    stage 0 (which makes no move, H1): cell 0's mean 50 is at squared distance 3*150^2 > tau^2
    -> y = -1; cell 1's mean 200 -> y = +1.  CLASS: only label 1 is active, so column 3 (label
    0, colour 200) never moves and the output keeps the wrong cut at x = 4 (no move at all:
    label 1's pixels gain nothing from the dark mean).  BSP (both superpixels touch the other
    class) and EQ7 (column 3's E neighbour has another label and class) keep H1's result."""
    p = params(2, [2, 1], 2, 65536, 32 * 65536, mask=rule, tau2=100, protos=[(200, 200, 200)])
    r = oracle.segment(_h1_image(), p)
    assert r.sp["y"].tolist() == [-1, 1]
    want = np.zeros((8, 8), dtype=np.int32)
    if rule == 1:
        want[:, 4:] = 1
        assert r.sp["active"].tolist() == [0, 1]
        assert r.counters[..., oracle.C_COMMIT].sum() == 0
    else:
        want[:, 3:] = 1
        assert r.counters[1, 0, :, oracle.C_COMMIT].tolist() == [0, 4, 0, 4]
    assert np.array_equal(r.labels[0], want)


def test_eq4_choice_is_brute_force_argmin_in_victim_order():
    """Every merge round of random MERGE runs, replayed by brute force from the pre-merge state
    and the exported victim flags: victims in ascending id; a locked victim is skipped; its
    target is the argmin over the 4-adjacent, alive, unlocked superpixels that pass Eq. 5
    ((n_T + n_A) u_den <= u_num InitSize_T) of the full per-pixel energy change of relabelling
    the whole victim (frozen means), lowest id on ties; no feasible target -> no merge.  The
    oracle's merge log must be exactly that sequence."""
    rng = np.random.default_rng(41)
    rounds = merges = skipped = 0
    for it in range(70):
        H, W = int(rng.integers(12, 19)), int(rng.integers(12, 19))
        img = cut_image(rng, H, W)
        M = 9
        sizes = [2, 1]
        lp, lb = int(rng.integers(0, 3 * 65536)), int(rng.integers(0, 40 * 65536))
        u = [(3, 2), (5, 4), (2, 1)][it % 3]
        p = params(M, sizes, 4, lp, lb, size_mode=2, u=u)
        geo = brute.geometry(H, W, M, sizes)
        full = oracle.segment(img, p, log_merges=1000)
        for s in range(len(sizes)):
            pre = oracle.segment(img, p, stop=(oracle.STOP_PHASE, s, p.sweeps - 1, 3))
            vict = [int(k) for k in np.nonzero(pre.victims)[0]]
            if not vict:
                continue
            rounds += 1
            xs, ys = geo[s]
            bmap, bsums, bsp = pre.map[0], brute.sp_sums(pre.sp), pre.sp
            pix = brute.expand(bmap, xs, ys)
            cq, mq = brute.quantised_means(bsums)
            E0 = brute.energy_int(img, pix, cq, mq, lp, lb)
            locked, want = set(), []
            for A in vict:
                if A in locked:
                    continue
                pa = pix == A
                adj = set()
                adj |= set(pix[:, 1:][pa[:, :-1]]) | set(pix[:, :-1][pa[:, 1:]])
                adj |= set(pix[1:, :][pa[:-1, :]]) | set(pix[:-1, :][pa[1:, :]])
                adj = {int(t) for t in adj} - {A}
                scores = []
                for T in sorted(adj):
                    if not bsp["alive"][T] or T in locked:
                        continue
                    if (bsums[T, 0] + bsums[A, 0]) * p.u_den > p.u_num * bsp["init_size"][T]:
                        continue
                    E1 = brute.energy_int(img, np.where(pix == A, T, pix), cq, mq, lp, lb)
                    scores.append((E1 - E0, T))
                if scores:
                    T = min(scores)[1]
                    want.append((A, T))
                    locked |= {A, T}
                else:
                    skipped += 1
            got = [(int(m["A"]), int(m["T"])) for m in full.merges if m["stage"] == s]
            assert got == want, (it, s, got, want)
            merges += len(want)
    assert rounds > 40 and merges > 40 and skipped > 0

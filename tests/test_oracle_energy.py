"""Pins for O6/O6' (Eqs. 1-3, E_topo, commit), O7 (Eqs. 4-5 merges), O8 (Eqs. 6-7) and
the hand-worked H1 case.  The brute-force side (tests/brute.py) recomputes Eq. 1 per pixel
from the label maps; nothing here calls the oracle's energy code.  -m "not gpu"."""
from fractions import Fraction
import copy

import numpy as np
import pytest

import oracle
import synth
import brute

F = 8
SCALE = 1 << (16 + 4 * F)  # oracle dE units: 2^(16+4F) x real energy


def params(M, sizes, sweeps, lam_pos=65536, lam_b=32 * 65536, size_mode=0, mask=0,
           l=(1, 4), u=(3, 2), tau2=1600, stats=0, protos=None):
    p = synth.Params(M, list(sizes), sweeps, lam_pos, lam_b, size_mode, l[0], l[1], u[0], u[1],
                     mask, protos if protos is not None else [synth.PROTO_PINK, synth.PROTO_PURPLE],
                     tau2, stats)
    return p


def cut_image(rng, H, W, noise=8):
    """piecewise-flat pink/purple/white image with 3 random straight cuts plus noise"""
    cols = np.array([synth.PROTO_PINK, synth.PROTO_PURPLE, (240, 235, 240), (70, 35, 100)])
    yy, xx = np.mgrid[0:H, 0:W]
    code = np.zeros((H, W), dtype=np.int64)
    for _ in range(3):
        a, b = rng.normal(size=2)
        c = rng.uniform(-1, 1) * (abs(a) * W + abs(b) * H) / 2
        code = code * 2 + ((a * (xx - W / 2) + b * (yy - H / 2) + c) > 0)
    pal = cols[rng.integers(0, 4, size=8)]
    img = pal[code].astype(np.int64) + rng.normal(0, noise, size=(H, W, 3)).round().astype(np.int64)
    return np.clip(img, 0, 255).astype(np.uint8)


def before_key(p, s, t, ph):
    if ph > 0:
        return (oracle.STOP_PHASE, s, t, ph - 1)
    if t > 0:
        return (oracle.STOP_PHASE, s, t - 1, 3)
    return (oracle.STOP_STAGE_START, s, 0, 0)


def state(img, p, key):
    r = oracle.segment(img, p, stop=key)
    assert r.dbg.stopped
    return r.map[0], brute.sp_sums(r.sp), r.sp


def dE_of(m):
    return oracle.i128(m["dE_hi"], m["dE_lo"])


# ---------------------------------------------------------------- H1
@pytest.mark.parametrize("lam_pos,lam_b", [(1, 32), (0, 0), (1000, 1000), (7, 0)])
def test_H1_hand_worked(lam_pos, lam_b):
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    img[:, 3:, :] = 200
    p = params(2, [2, 1], 2, lam_pos * 65536, lam_b * 65536)
    r = oracle.segment(img, p, log_moves=100)
    commits = r.counters[:2, :2, :, oracle.C_COMMIT]
    assert commits[0].tolist() == [[0, 0, 0, 0], [0, 0, 0, 0]]
    assert commits[1].tolist() == [[0, 4, 0, 4], [0, 0, 0, 0]]
    want = np.zeros((8, 8), dtype=np.int32)
    want[:, 3:] = 1
    assert np.array_equal(r.labels[0], want)
    sums = brute.sp_sums(r.sp)
    assert sums[0].tolist() == [24, 0, 0, 0, 24, 84]
    assert sums[1].tolist() == [40, 8000, 8000, 8000, 200, 140]
    mv = {(int(m["bi"]), int(m["bj"])): m for m in r.moves}
    assert sorted(mv) == [(3, y) for y in range(8)]
    # (3,0): dC = -3*150^2, dP = +4, dB2 = +2 (top border) in real units
    assert dE_of(mv[(3, 0)]) == SCALE * (-67500 + 4 * lam_pos + 2 * lam_b)
    # (3,2): dP = +4, dB2 = +4
    assert dE_of(mv[(3, 2)]) == SCALE * (-67500 + 4 * lam_pos + 4 * lam_b)
    assert all(mv[(3, y)]["phase"] == (1 if y % 2 == 0 else 3) for y in range(8))


def test_H1_intermediate_snapshot():
    img = np.zeros((8, 8, 3), dtype=np.uint8)
    img[:, 3:, :] = 200
    p = params(2, [2, 1], 2)
    _, sums, _ = state(img, p, (oracle.STOP_PHASE, 1, 0, 1))
    assert sums[0].tolist() == [28, 800, 800, 800, 36, 100]
    assert sums[1].tolist() == [36, 7200, 7200, 7200, 188, 124]
    assert oracle.round_mean(800, 28) == 7314  # c0 ~ 28.57


# ---------------------------------------------------------------- O6 brute force
def _random_cases(n, seed, sizes_choices=((2, 1), (4, 2, 1)), block_aligned=False):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        H, W = int(rng.integers(8, 17)), int(rng.integers(8, 17))
        if block_aligned:
            H, W = H - H % 4, W - W % 4
        M = int(rng.integers(2, 10))
        try:
            oracle.grid(H, W, M)
        except oracle.OracleError:
            continue
        if rng.random() < 0.5:
            img = cut_image(rng, H, W)
        else:
            img = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
        sizes = list(sizes_choices[int(rng.integers(len(sizes_choices)))])
        lam_pos = int(rng.integers(0, 5 * 65536))
        lam_b = int(rng.integers(0, 64 * 65536))
        yield img, H, W, M, sizes, lam_pos, lam_b, rng


def test_move_dE_equals_brute_force_energy_difference():
    """Every committed move's dE == E(after that single move) - E(before) with the frozen
    quantised means, per pixel (Eq. 1 + Eq. 2), exactly; and the phase's moves add up (A6)."""
    checked = 0
    for img, H, W, M, sizes, lp, lb, rng in _random_cases(14, 2):
        p = params(M, sizes, 2, lp, lb)
        geo = brute.geometry(H, W, M, sizes)
        full = oracle.segment(img, p, log_moves=100000)
        for s in range(len(sizes)):
            xs, ys = geo[s]
            for t in range(p.sweeps):
                for ph in range(4):
                    mv = [m for m in full.moves if (m["stage"], m["sweep"], m["phase"]) == (s, t, ph)]
                    if not mv:
                        continue
                    bmap, bsums, _ = state(img, p, before_key(p, s, t, ph))
                    amap, _, _ = state(img, p, (oracle.STOP_PHASE, s, t, ph))
                    cq, mq = brute.quantised_means(bsums)
                    pix0 = brute.expand(bmap, xs, ys)
                    E0 = brute.energy_int(img[0] if img.ndim == 4 else img, pix0, cq, mq, lp, lb)
                    total = 0
                    for m in mv:
                        one = bmap.copy()
                        assert one[m["bj"], m["bi"]] == m["A"]
                        one[m["bj"], m["bi"]] = m["B"]
                        E1 = brute.energy_int(img, brute.expand(one, xs, ys), cq, mq, lp, lb)
                        assert E1 - E0 == dE_of(m)
                        assert dE_of(m) < 0
                        total += dE_of(m)
                        checked += 1
                    Ea = brute.energy_int(img, brute.expand(amap, xs, ys), cq, mq, lp, lb)
                    assert Ea - E0 == total
    assert checked > 200


def test_phase_invariants_all_size_modes():
    """After every phase: every label 4-connected; sums == recount; alive count never grows;
    HARD/MERGE keep n*l_den >= l_num*InitSize (A19); only phase-colour blocks changed."""
    for img, H, W, M, sizes, lp, lb, rng in _random_cases(10, 3):
        geo = brute.geometry(H, W, M, sizes)
        for mode in (0, 1, 2):
            p = params(M, sizes, 2, lp, lb, size_mode=mode)
            prev_alive = M
            for s in range(len(sizes)):
                xs, ys = geo[s]
                prev = None
                for t in range(p.sweeps):
                    for ph in range(4):
                        bmap, sums, sp = state(img, p, (oracle.STOP_PHASE, s, t, ph))
                        pix = brute.expand(bmap, xs, ys)
                        assert brute.all_connected(pix)
                        assert np.array_equal(brute.recount(img, pix, M), sums)
                        alive = int(sp["alive"].sum())
                        assert alive == len(np.unique(bmap)) and alive <= prev_alive
                        prev_alive = alive
                        if mode:
                            a = sp["alive"] == 1
                            assert np.all(sums[a, 0] * p.l_den >= p.l_num * sp["init_size"][a])
                        if prev is not None:
                            jj, ii = np.nonzero(prev != bmap)
                            assert np.all(ii % 2 == (ph & 1)) and np.all(jj % 2 == (ph >> 1))
                        prev = bmap


def test_descent_within_rounding_slack():
    """E_real (exact means) after a phase <= before + sum(dE_real) + N(3+2 lam_pos)2^(-2F-2) (A29)."""
    for img, H, W, M, sizes, lp, lb, rng in _random_cases(8, 4):
        p = params(M, sizes, 2, lp, lb)
        geo = brute.geometry(H, W, M, sizes)
        full = oracle.segment(img, p, log_moves=100000)
        lam_pos, lam_b = Fraction(lp, 65536), Fraction(lb, 65536)
        slack = H * W * (3 + 2 * lam_pos) * Fraction(1, 2 ** (2 * F + 2))
        for s in range(len(sizes)):
            xs, ys = geo[s]
            for t in range(p.sweeps):
                for ph in range(4):
                    mv = [m for m in full.moves if (m["stage"], m["sweep"], m["phase"]) == (s, t, ph)]
                    bmap, _, _ = state(img, p, before_key(p, s, t, ph))
                    amap, _, _ = state(img, p, (oracle.STOP_PHASE, s, t, ph))
                    e0 = brute.energy_real(img, brute.expand(bmap, xs, ys), lam_pos, lam_b)
                    e1 = brute.energy_real(img, brute.expand(amap, xs, ys), lam_pos, lam_b)
                    d = sum(Fraction(dE_of(m), SCALE) for m in mv)
                    assert e1 <= e0 + d + slack


# ---------------------------------------------------------------- O7 merges (Eqs. 4-5)
def test_merge_round_brute_force():
    merges_checked = 0
    rng = np.random.default_rng(5)
    for it in range(60):
        H, W = int(rng.integers(12, 19)), int(rng.integers(12, 19))
        img = cut_image(rng, H, W)
        M = 9
        sizes = [2, 1]
        lp, lb = int(rng.integers(0, 3 * 65536)), int(rng.integers(0, 40 * 65536))
        p = params(M, sizes, 4, lp, lb, size_mode=2)
        geo = brute.geometry(H, W, M, sizes)
        full = oracle.segment(img, p, log_merges=1000)
        for s in range(len(sizes)):
            mg = [m for m in full.merges if m["stage"] == s]
            if not mg:
                continue
            xs, ys = geo[s]
            bmap, bsums, bsp = state(img, p, (oracle.STOP_PHASE, s, p.sweeps - 1, 3))
            amap, asums, asp = state(img, p, (oracle.STOP_AFTER_MERGE, s, 0, 0))
            cq, mq = brute.quantised_means(bsums)
            pix0 = brute.expand(bmap, xs, ys)
            E0 = brute.energy_int(img, pix0, cq, mq, lp, lb)
            used = set()
            for m in mg:
                A, T = int(m["A"]), int(m["T"])
                assert A not in used and T not in used  # locks (O7 step 4)
                used |= {A, T}
                one = np.where(bmap == A, T, bmap)
                E1 = brute.energy_int(img, brute.expand(one, xs, ys), cq, mq, lp, lb)
                assert E1 - E0 == dE_of(m)
                # shared edge length
                pa = pix0 == A
                pt = pix0 == T
                e = int(np.count_nonzero(pa[:, 1:] & pt[:, :-1]) + np.count_nonzero(pa[:, :-1] & pt[:, 1:]) +
                        np.count_nonzero(pa[1:, :] & pt[:-1, :]) + np.count_nonzero(pa[:-1, :] & pt[1:, :]))
                assert e == m["len"] > 0
                # Eq. 5 upper bound
                assert (bsums[T, 0] + bsums[A, 0]) * p.u_den <= p.u_num * bsp["init_size"][T]
                merges_checked += 1
            pix1 = brute.expand(amap, xs, ys)
            assert brute.all_connected(pix1)
            assert np.array_equal(brute.recount(img, pix1, M), asums)
            assert int(asp["alive"].sum()) == int(bsp["alive"].sum()) - len(mg)
            assert np.array_equal(asp["init_size"], bsp["init_size"])
    assert merges_checked > 20


# ---------------------------------------------------------------- special cases
def test_single_superpixel_and_constant_image_make_no_moves():
    rng = np.random.default_rng(6)
    img = rng.integers(0, 256, size=(20, 24, 3), dtype=np.uint8)
    r = oracle.segment(img, params(1, [4, 2, 1], 3))
    assert r.counters[..., oracle.C_CAND].sum() == 0 and np.all(r.labels == 0)
    const = np.full((32, 48, 3), 123, dtype=np.uint8)
    for M in (6, 24):
        for mode in (0, 1, 2):
            r = oracle.segment(const, params(M, [8, 4, 2, 1], 3, size_mode=mode))
            assert r.counters[..., oracle.C_COMMIT].sum() == 0
            assert r.counters[..., oracle.C_CAND].sum() > 0


def test_size_modes_agree_when_no_gate_can_fire_and_recount_equals_reuse():
    for img, H, W, M, sizes, lp, lb, rng in _random_cases(8, 7):
        outs = []
        for mode in (0, 1, 2):
            r = oracle.segment(img, params(M, sizes, 3, lp, lb, size_mode=mode, l=(0, 4)))
            outs.append(r.labels)
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
        for mode in (0, 2):
            a = oracle.segment(img, params(M, sizes, 3, lp, lb, size_mode=mode, stats=0))
            b = oracle.segment(img, params(M, sizes, 3, lp, lb, size_mode=mode, stats=1))
            assert np.array_equal(a.labels, b.labels) and np.array_equal(a.sp, b.sp)


def test_batch_equals_singles():
    w = synth.scaled(5, 64, 80, B=3)
    img = w.images()
    r = oracle.segment(img, w.params)
    M = w.params.n_superpixels
    for b in range(3):
        s = oracle.segment(img[b], w.params)
        assert np.array_equal(r.labels[b], s.labels[0])
        assert np.array_equal(r.sp[b * M:(b + 1) * M], s.sp)


# ---------------------------------------------------------------- O8 prediction
def test_prediction_closed_cases():
    H, W = 32, 64
    img = np.zeros((H, W, 3), dtype=np.uint8)
    img[:, :32] = synth.PROTO_PINK
    img[:, 32:] = (240, 235, 240)
    sizes = [8, 4, 2, 1]
    for rule in (1, 2, 3):
        p = params(8, sizes, 2, mask=rule, tau2=400)
        r = oracle.segment(img, p, stop=(oracle.STOP_AFTER_PREDICT, 0, 0, 0))
        sp = r.sp
        # grid 2x4 of 16x16 cells; columns 0,1 pink (d=0 -> y=+1), 2,3 white (d=5925 -> y=-1)
        assert sp["y"].tolist() == [1, 1, -1, -1] * 2
        if rule == 1:
            assert sp["active"].tolist() == [1, 1, 0, 0] * 2
        else:  # boundary superpixels: the two columns touching the pink/white border
            assert sp["active"].tolist() == [0, 1, 1, 0] * 2
    # tau2 boundary case of Eq. 6: d == tau^2 -> h = 0 -> y = +1
    img2 = np.full((16, 16, 3), 0, dtype=np.uint8)
    img2[...] = (230 + 20, 170, 200)  # distance^2 to pink = 400
    p = params(1, [4, 1], 1, mask=1, tau2=400)
    assert oracle.segment(img2, p, stop=(oracle.STOP_AFTER_PREDICT, 0, 0, 0)).sp["y"][0] == 1
    p = params(1, [4, 1], 1, mask=1, tau2=399)
    assert oracle.segment(img2, p, stop=(oracle.STOP_AFTER_PREDICT, 0, 0, 0)).sp["y"][0] == -1


def test_mask_rules_restrict_candidates():
    """tau huge + CLASS == OFF; all y equal -> BSP/EQ7 freeze later stages;
    candidates EQ7 <= BSP <= OFF from the same state ("strengthen the restriction")."""
    w = synth.scaled(3, 96, 128)
    img = w.images()
    base = copy.deepcopy(w.params)
    base.size_mode = 0
    off = copy.deepcopy(base); off.mask_rule = 0
    r_off = oracle.segment(img, off)
    huge = copy.deepcopy(base); huge.mask_rule = 1; huge.tau2 = 10 ** 9
    r_huge = oracle.segment(img, huge)
    assert np.array_equal(r_off.labels, r_huge.labels)
    for rule in (2, 3):
        q = copy.deepcopy(base); q.mask_rule = rule; q.tau2 = 10 ** 9
        r = oracle.segment(img, q)
        assert r.counters[1:, :, :, oracle.C_COMMIT].sum() == 0
    cands = {}
    for rule in (0, 2, 3):
        q = copy.deepcopy(base); q.mask_rule = rule
        r = oracle.segment(img, q)
        cands[rule] = r.counters[1, 0, 0, oracle.C_CAND]
    assert cands[3] <= cands[2] <= cands[0]


def test_block_move_matches_full_phase():
    """orc_block_move (used for sampled checks at full scale) reproduces a whole phase of the
    oracle: from the state before phase (s,t,ph), every block of the phase colour moves exactly
    as in the full run (NONE, mask OFF)."""
    w = synth.config(1)
    img = w.images()[0]
    p = copy.deepcopy(w.params)
    geo = brute.geometry(w.H, w.W, p.n_superpixels, p.block_sizes)
    checked = moved = 0
    for (s, t, ph) in [(4, 0, 1), (4, 1, 2), (3, 0, 3)]:
        bmap, sums, _ = state(img, p, before_key(p, s, t, ph))
        amap, _, _ = state(img, p, (oracle.STOP_PHASE, s, t, ph))
        xs, ys = geo[s]
        cq, mq = brute.quantised_means(sums)
        H, W = bmap.shape
        for j in range(ph >> 1, H, 2):
            for i in range(ph & 1, W, 2):
                win = np.full(9, -1, dtype=np.int32)
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        if 0 <= i + dx < W and 0 <= j + dy < H:
                            win[(dy + 1) * 3 + dx + 1] = bmap[j + dy, i + dx]
                means = np.zeros((9, 5), dtype=np.int64)
                for c in range(9):
                    if win[c] >= 0:
                        means[c] = [*cq[win[c]], *mq[win[c]]]
                x0, x1, y0, y1 = xs[i], xs[i + 1], ys[j], ys[j + 1]
                blk = img[y0:y1, x0:x1].reshape(-1, 3).astype(np.int64)
                yy, xx = np.mgrid[y0:y1, x0:x1]
                d = [blk.shape[0], *blk.sum(0), int(xx.sum()), int(yy.sum())]
                e = [x1 - x0, y1 - y0, x1 - x0, y1 - y0]
                code, B, dE = oracle.block_move(win, means, d, e, p)
                want = B if code == 3 else bmap[j, i]
                assert amap[j, i] == want, (s, t, ph, i, j)
                checked += 1
                moved += code == 3
    assert moved > 50 and checked > 5000

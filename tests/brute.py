"""Test-side brute-force checkers, written from the paper's definitions and independent
of the oracle's code: per-pixel energy (Eq. 1 with Eq. 2), exact rational means,
flood-fill connectivity, recounts.  Used to pin the oracle (tests -m "not gpu")."""
from __future__ import annotations

from fractions import Fraction
import math

import numpy as np
from scipy import ndimage

import oracle

F = 8
FOUR = np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]])


def round_half_up(fr: Fraction) -> int:
    return math.floor(fr + Fraction(1, 2))


def geometry(H, W, M, block_sizes):
    """Per-stage (xs, ys) via the oracle's O1/O2 functions (pinned in test_oracle_geometry)."""
    r, c = oracle.grid(H, W, M)
    X = [(i * W) // c for i in range(c + 1)]
    Y = [(j * H) // r for j in range(r + 1)]
    return [(oracle.stage_axis(W, b, X), oracle.stage_axis(H, b, Y)) for b in block_sizes]


def expand(block_map, xs, ys):
    """block map [nby][nbx] -> pixel map [H][W]"""
    return np.repeat(np.repeat(block_map, np.diff(ys), axis=0), np.diff(xs), axis=1)


def recount(img, pixmap, M):
    """int64 sums {n, r, g, b, x, y} per label from a pixel label map."""
    H, W = pixmap.shape
    lab = pixmap.ravel()
    yy, xx = np.mgrid[0:H, 0:W]
    out = np.zeros((M, 6), dtype=np.int64)
    out[:, 0] = np.bincount(lab, minlength=M)
    for ch in range(3):
        out[:, 1 + ch] = np.bincount(lab, weights=img[..., ch].ravel().astype(np.float64), minlength=M).astype(np.int64)
    out[:, 4] = np.bincount(lab, weights=xx.ravel().astype(np.float64), minlength=M).astype(np.int64)
    out[:, 5] = np.bincount(lab, weights=yy.ravel().astype(np.float64), minlength=M).astype(np.int64)
    return out


def sp_sums(sp):
    return np.stack([sp["n"], sp["sum_r"], sp["sum_g"], sp["sum_b"], sp["sum_x"], sp["sum_y"]], axis=1)


def quantised_means(sums):
    """cq[k][3], mq[k][2] = round-half-up(2^F * mean) with exact rationals (A24)."""
    M = sums.shape[0]
    cq = np.zeros((M, 3), dtype=object)
    mq = np.zeros((M, 2), dtype=object)
    for k in range(M):
        n = int(sums[k, 0])
        if n <= 0:
            continue
        for ch in range(3):
            cq[k, ch] = round_half_up(Fraction(int(sums[k, 1 + ch]) << F, n))
        for d in range(2):
            mq[k, d] = round_half_up(Fraction(int(sums[k, 4 + d]) << F, n))
    return cq, mq


def energy_int(img, pixmap, cq, mq, lam_pos_q16, lam_b_q16):
    """2^(16+4F) x Eq. 1 (without E_topo / E_size) under the given quantised means:
    W_c sum_p ||2^F I_p - cq||^2 + W_p sum_p ||2^F p - mq||^2 + W_b sum_p sum_{q in N4} [s_p != s_q]."""
    H, W = pixmap.shape
    col = 0
    pos = 0
    labels = np.unique(pixmap)
    yy, xx = np.mgrid[0:H, 0:W]
    for k in labels:
        m = pixmap == k
        for ch in range(3):
            v = (img[..., ch][m].astype(object) << F) - cq[k, ch]
            col += int(sum(int(t) * int(t) for t in v))
        for d, coord in enumerate((xx, yy)):
            v = (coord[m].astype(object) << F) - mq[k, d]
            pos += int(sum(int(t) * int(t) for t in v))
    bnd = 0
    bnd += 2 * int(np.count_nonzero(pixmap[:, 1:] != pixmap[:, :-1]))
    bnd += 2 * int(np.count_nonzero(pixmap[1:, :] != pixmap[:-1, :]))
    return (col << (2 * F + 16)) + (lam_pos_q16 << (2 * F)) * pos + (lam_b_q16 << (4 * F)) * bnd


def energy_real(img, pixmap, lam_pos, lam_b):
    """Eq. 1 (E_col + lam_pos E_pos + lam_b E_b) with EXACT means, as a Fraction."""
    H, W = pixmap.shape
    yy, xx = np.mgrid[0:H, 0:W]
    E = Fraction(0)
    for k in np.unique(pixmap):
        m = pixmap == k
        n = int(m.sum())
        for arr, w in [(img[..., 0], 1), (img[..., 1], 1), (img[..., 2], 1), (xx, lam_pos), (yy, lam_pos)]:
            v = arr[m].astype(np.int64)
            s, s2 = int(v.sum()), int((v * v).sum())
            E += w * (Fraction(s2) - Fraction(s * s, n))  # sum (v - mean)^2
    bnd = 2 * int(np.count_nonzero(pixmap[:, 1:] != pixmap[:, :-1])) + \
        2 * int(np.count_nonzero(pixmap[1:, :] != pixmap[:-1, :]))
    return E + lam_b * bnd


def all_connected(pixmap):
    """every label present is one 4-connected component"""
    for k in np.unique(pixmap):
        _, n = ndimage.label(pixmap == k, structure=FOUR)
        if n != 1:
            return False
    return True


def local_simple(mask):
    """Flood-fill definition: with p removed, the ring positions equal to A (bit k of mask,
    k = N,NE,E,SE,S,SW,W,NW) that are 4-adjacent to p (N,E,S,W) are all 4-connected to each
    other inside the 3x3 window, using only A positions of the window other than p."""
    pos = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]
    cells = {pos[k] for k in range(8) if (mask >> k) & 1}
    edge = [c for c in [(0, -1), (1, 0), (0, 1), (-1, 0)] if c in cells]
    if not edge:
        return False  # p is isolated from A: removing it empties / disconnects nothing local
    seen = {edge[0]}
    stack = [edge[0]]
    while stack:
        x, y = stack.pop()
        for dx, dy in [(0, 1), (1, 0), (0, -1), (-1, 0)]:
            q = (x + dx, y + dy)
            if q in cells and q not in seen:
                seen.add(q)
                stack.append(q)
    return all(e in seen for e in edge)

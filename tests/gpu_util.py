"""Helpers for the -m gpu parity tests: run the CUDA path (through the C ABI) and the oracle on
the same seeded input and compare element by element."""
from __future__ import annotations

import numpy as np

import oracle

CMP_FIELDS = ("n", "sum_r", "sum_g", "sum_b", "sum_x", "sum_y", "init_size", "alive")


def gpu_run(rapid, img, params):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img if img.ndim == 4 else img[None])).cuda()
    lab = rapid.segment(t, params)
    torch.cuda.synchronize()
    B = t.shape[0]
    sp, info = rapid.stats(B * params.n_superpixels)
    return lab.cpu().numpy(), sp, info


def first_divergence(rapid, img, params):
    """Bisect (stage, sweep, phase) stop points for the first map difference."""
    import torch
    img4 = img if img.ndim == 4 else img[None]
    t = torch.from_numpy(np.ascontiguousarray(img4)).cuda()
    B, H, W, _ = img4.shape
    points = []
    for s in range(len(params.block_sizes)):
        points.append((oracle.STOP_STAGE_START, s, 0, 0))
        for sw in range(params.sweeps):
            for ph in range(4):
                points.append((oracle.STOP_PHASE, s, sw, ph))
        points.append((oracle.STOP_AFTER_MERGE, s, 0, 0))
    cap = B * (H + 2) * (W + 2) * 2
    for pt in points:
        o = oracle.segment(img4, params, stop=pt, map_cap=cap)
        rapid.debug_stop(*pt)
        rapid.segment(t, params)
        torch.cuda.synchronize()
        g = rapid.debug_map(cap)
        rapid.debug_stop(0)
        if o.map is None or g.shape != o.map.shape or not np.array_equal(g, o.map):
            if o.map is not None and g.shape == o.map.shape:
                idx = np.argwhere(g != o.map)[:5].tolist()
                return f"first divergence at {pt}: {idx} gpu={[int(g[tuple(i)]) for i in idx]} " \
                       f"oracle={[int(o.map[tuple(i)]) for i in idx]}"
            return f"first divergence at {pt}: shapes {g.shape} vs {None if o.map is None else o.map.shape}"
    return "no map divergence found at stop points (stats/final only)"


def assert_parity(rapid, img, params, check_counters=True, diagnose=True):
    img4 = img if img.ndim == 4 else img[None]
    o = oracle.segment(img4, params)
    g_lab, g_sp, info = gpu_run(rapid, img4, params)
    ok = np.array_equal(g_lab, o.labels)
    if not ok and diagnose:
        raise AssertionError(f"labels differ ({int((g_lab != o.labels).sum())} px); "
                             + first_divergence(rapid, img4, params))
    assert ok, "labels differ"
    for f in CMP_FIELDS:
        assert np.array_equal(g_sp[f].astype(np.int64), o.sp[f].astype(np.int64)), f
    if params.mask_rule != 0:
        assert np.array_equal(g_sp["y"], o.sp["y"]), "y"
        alive = o.sp["alive"] == 1
        assert np.array_equal(g_sp["active"][alive], o.sp["active"][alive]), "active"
    # derived float means within 1e-6 relative of the exact ratio
    n = o.sp["n"].astype(np.float64)
    nz = n > 0
    for f, m in (("sum_r", "mean_r"), ("sum_x", "mean_x"), ("sum_y", "mean_y")):
        want = o.sp[f][nz] / n[nz]
        assert np.all(np.abs(g_sp[m][nz] - want) <= 1e-6 * np.maximum(1.0, np.abs(want)))
    if check_counters:
        gc = info.counters()
        oc = o.counters
        assert np.array_equal(gc[..., oracle.C_COMMIT], oc[..., oracle.C_COMMIT]), "commits per phase"
        ns = len(params.block_sizes)
        for s in range(ns):
            run = info.stage_sweeps_run[s]
            assert np.array_equal(gc[s, :run], oc[s, :run]), f"counters stage {s}"
        assert list(info.stage_merges)[:ns] == o.stage_merges[:ns]
        assert list(info.stage_victims)[:ns] == o.stage_victims[:ns]
    return o, g_lab, g_sp, info

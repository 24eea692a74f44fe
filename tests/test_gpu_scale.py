"""Config 4 at full size (32768^2 = 1.07 Gpx, M = 2^20) in the launch configuration bench.py
times.  The whole oracle cannot run at this size in a test, so parity is checked
(a) on sampled outputs the oracle computes one by one (orc_block_move, pinned against full
    oracle phases in test_oracle_energy.py) from a GPU state stopped mid-stage, and
(b) via properties that hold at any size: determinism, int64 sums == recount of the label map,
    alive superpixels == distinct labels, every superpixel 4-connected, size floor (MERGE)."""
import copy

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cfg4():
    import torch
    import paper_1704_02083_b200 as rb
    w = synth.config(4)
    host = torch.empty((w.B, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
    w.images(out=host.numpy())
    img = host.cuda()
    r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=w.B * w.params.n_superpixels)
    yield w, host, img, r
    r.close()


def recount(lab, img, M):
    """int64 sums {n, r, g, b, x, y} per label from the label map (torch on the GPU, float64
    bincount is exact below 2^53)."""
    import torch
    H, W = lab.shape[-2:]
    flat = lab.reshape(-1).long()
    out = [torch.bincount(flat, minlength=M).double()]
    for ch in range(3):
        out.append(torch.bincount(flat, weights=img[..., ch].reshape(-1).double(), minlength=M))
    xs = torch.arange(W, device=lab.device, dtype=torch.float64).expand(H, W).reshape(-1)
    ys = torch.arange(H, device=lab.device, dtype=torch.float64).view(H, 1).expand(H, W).reshape(-1)
    out.append(torch.bincount(flat, weights=xs, minlength=M))
    out.append(torch.bincount(flat, weights=ys, minlength=M))
    return torch.stack(out, 1).round().long().cpu().numpy()


def n_components(lab):
    """number of 4-connected components of equal labels (min-label propagation + pointer
    jumping on the GPU)"""
    import torch
    H, W = lab.shape
    comp = torch.arange(H * W, device=lab.device, dtype=torch.int32).view(H, W)
    big = torch.iinfo(torch.int32).max
    for _ in range(100000):
        new = comp.clone()
        eqh = lab[:, 1:] == lab[:, :-1]
        eqv = lab[1:, :] == lab[:-1, :]
        new[:, 1:] = torch.minimum(new[:, 1:], torch.where(eqh, comp[:, :-1], big))
        new[:, :-1] = torch.minimum(new[:, :-1], torch.where(eqh, comp[:, 1:], big))
        new[1:, :] = torch.minimum(new[1:, :], torch.where(eqv, comp[:-1, :], big))
        new[:-1, :] = torch.minimum(new[:-1, :], torch.where(eqv, comp[1:, :], big))
        flat = new.view(-1)
        new = flat[flat.long()].view(H, W)  # pointer jumping
        if torch.equal(new, comp):
            break
        comp = new
    roots = (comp.view(-1) == torch.arange(H * W, device=lab.device, dtype=torch.int32)).sum()
    return int(roots)


def test_config4_full_size_properties(cfg4):
    import torch
    w, host, img, r = cfg4
    p = w.params
    M = p.n_superpixels
    lab1 = r.segment(img, p)
    torch.cuda.synchronize()
    sp, info = r.stats(M)
    lab2 = r.segment(img, p)
    torch.cuda.synchronize()
    assert torch.equal(lab1, lab2)  # deterministic
    lab = lab1[0]
    sums = np.stack([sp[f] for f in ("n", "sum_r", "sum_g", "sum_b", "sum_x", "sum_y")], 1)
    assert np.array_equal(recount(lab, img[0], M), sums)
    alive = sp["alive"] == 1
    assert int(alive.sum()) == int(torch.unique(lab).numel()) == int(info.alive)
    assert np.all(sums[alive, 0] * p.l_den >= p.l_num * sp["init_size"][alive])  # A19 floor
    assert np.all(sums[~alive, 0] == 0)
    del lab2
    torch.cuda.empty_cache()
    assert n_components(lab) == int(alive.sum())  # every superpixel 4-connected
    assert 0 < info.active < info.alive
    assert sum(info.stage_merges[:6]) > 0


def test_config4_sampled_block_decisions_match_oracle(cfg4):
    """Stop the full-size run before and after one pixel-stage phase (size_mode NONE so every
    proposal commits, mask on) and recompute sampled blocks of the phase colour with the
    oracle's per-block decision from the GPU's pre-phase state."""
    import torch
    w, host, img, r = cfg4
    p = copy.deepcopy(w.params)
    p.size_mode = synth.SIZE_NONE
    M = p.n_superpixels
    s, t, ph = len(p.block_sizes) - 1, 0, 1
    cap = w.pixels + 16
    r.debug_stop(oracle.STOP_PHASE, s, t, ph - 1)
    r.segment(img, p)
    torch.cuda.synchronize()
    before = r.debug_map(cap)[0]
    sp, _ = r.stats(M)
    r.debug_stop(oracle.STOP_PHASE, s, t, ph)
    r.segment(img, p)
    torch.cuda.synchronize()
    after = r.debug_map(cap)[0]
    r.debug_stop(0)
    H, W = before.shape
    im = host.numpy()[0]
    rng = np.random.default_rng(0)
    # sample boundary-rich positions: blocks of the phase colour whose label changed plus random ones
    ys, xs = np.nonzero(before != after)
    assert len(ys) > 1000
    pick = rng.choice(len(ys), size=4000, replace=False)
    cand = list(zip(ys[pick], xs[pick]))
    for _ in range(4000):
        cand.append((2 * int(rng.integers(1, H // 2 - 1)) + (ph >> 1), 2 * int(rng.integers(1, W // 2 - 1)) + (ph & 1)))
    means_of = {}
    moved = 0
    for (y, x) in cand:
        assert y % 2 == (ph >> 1) and x % 2 == (ph & 1)
        win = np.full(9, -1, dtype=np.int32)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if 0 <= y + dy < H and 0 <= x + dx < W:
                    win[(dy + 1) * 3 + dx + 1] = before[y + dy, x + dx]
        means = np.zeros((9, 5), dtype=np.int64)
        for c in range(9):
            l = int(win[c])
            if l < 0:
                continue
            if l not in means_of:
                n = int(sp["n"][l])
                means_of[l] = ([oracle.colour_mean(int(sp[f][l]), n) for f in ("sum_r", "sum_g", "sum_b")]
                               + [oracle.round_mean(int(sp[f][l]), n) for f in ("sum_x", "sum_y")])
            means[c] = means_of[l]
        d = [1, int(im[y, x, 0]), int(im[y, x, 1]), int(im[y, x, 2]), x, y]
        code, B, _ = oracle.block_move(win, means, d, [1, 1, 1, 1], p)
        A = int(before[y, x])
        gate = sp["active"][A] == 1  # CLASS mask after prediction (A22)
        want = B if (code == 3 and gate) else A
        assert int(after[y, x]) == want, (y, x, code, A, B)
        moved += want != A
    assert moved >= 4000


def test_config4_full_size_bit_exact_with_oracle(cfg4):
    """North-star target #1 at the headline size: the whole config-4 segmentation (1.07 Gpx,
    M = 2^20, MERGE + CLASS + REUSE, stages 32..1 incl. the 64-bit b = 16 stage) on the GPU, in
    the launch configuration bench.py times (CUDA-graph replay), against the single-threaded
    CPU oracle on the same input: labels, int64 sums, flags and every per-phase counter
    element by element (oracle ~2-3 min and ~30 GB of host RAM)."""
    import time
    import torch
    from gpu_util import CMP_FIELDS
    w, host, img, r = cfg4
    p = w.params
    M = p.n_superpixels
    labels = torch.empty((1, w.H, w.W), dtype=torch.int32, device="cuda")
    r.segment(img, p, labels)  # capture
    r.segment(img, p, labels)  # replay (the timed launch configuration)
    torch.cuda.synchronize()
    sp, info = r.stats(M)
    g_lab = labels.cpu().numpy()
    del labels
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    o = oracle.segment(host.numpy(), p)
    dt = time.perf_counter() - t0
    print(f"\nconfig 4 oracle: {dt:.1f} s ({w.pixels / dt / 1e6:.2f} Mpx/s, 1 thread)")
    diff = int((g_lab != o.labels).sum())
    assert diff == 0, f"{diff} labels differ"
    for f in CMP_FIELDS + ("y",):
        assert np.array_equal(sp[f].astype(np.int64), o.sp[f].astype(np.int64)), f
    alive = o.sp["alive"] == 1
    assert np.array_equal(sp["active"][alive], o.sp["active"][alive]), "active"
    gc, oc = info.counters(), o.counters
    for s in range(len(p.block_sizes)):
        run = int(info.stage_sweeps_run[s])
        assert np.array_equal(gc[s, :run], oc[s, :run]), f"per-phase counters, stage {s}"
    assert list(info.stage_merges)[:6] == o.stage_merges[:6]
    assert list(info.stage_victims)[:6] == o.stage_victims[:6]
    assert o.counters[1, ..., oracle.C_COMMIT].sum() > 10000  # the 64-bit b = 16 stage moves blocks

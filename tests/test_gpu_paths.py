"""GPU: the launch and sweep variants of the library give identical results (and match the
oracle): boundary-set sweep replayed from a CUDA graph (default), the same enqueued kernel by
kernel (RAPID_NO_GRAPH=1), and the full-scan sweep K4a + K4b (RAPID_SWEEP=scan), which shares
no candidate-selection code with the boundary-set path.  Also: replaying a captured graph
after changing the image contents in place, and after changing parameters."""
import copy
import os

import numpy as np
import pytest

import oracle
import synth
from gpu_util import gpu_run

pytestmark = pytest.mark.gpu


def make_ctx(env, pixels, sps):
    import paper_1704_02083_b200 as rb
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return rb.Rapid(0, max_pixels=pixels, max_superpixels=sps)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


VARIANTS = [{}, {"RAPID_NO_GRAPH": "1"}, {"RAPID_SWEEP": "scan"}, {"RAPID_FUSE_BSET": "1"}, {"RAPID_FUSE_SNAP": "1"},
            {"RAPID_NO_TMA": "1"}, {"RAPID_BSET_PARENT": "0"}, {"RAPID_SWEEP_NO_SMALLB": "1"},
            {"RAPID_PDL": "1"}, {"RAPID_ADJ": "tma"}, {"RAPID_BSET_ROWS": "0"},
            {"RAPID_BSET_ROWS": "2"}, {"RAPID_PACKED": "1"},
            {"RAPID_SWEEP_LIST": "2"}, {"RAPID_ADJ_ILP": "4"}, {"RAPID_ADJ_ILP": "2"}, {"RAPID_ADJ_MINB8": "0"}, {"RAPID_SWEEP_UNI": "0"}]


@pytest.mark.parametrize("cfg,side", [(2, 1024), (4, 1024), (5, 0)])
def test_variants_identical_and_oracle_exact(cfg, side):
    w = synth.scaled(cfg, side, side) if side else synth.config(cfg)
    if cfg == 5:  # a 4-image batch of config 5 (independent tiles, distinct seeds)
        w.seeds, w.regions, w.nuclei, w.B = w.seeds[:4], w.regions[:4], w.nuclei[:4], 4
    img = w.images()
    ref = oracle.segment(img, w.params)
    outs = []
    for env in VARIANTS:
        r = make_ctx(env, w.pixels, w.B * w.params.n_superpixels)
        try:
            lab, sp, info = gpu_run(r, img, w.params)
        finally:
            r.close()
        assert np.array_equal(lab, ref.labels), f"{env}: {int((lab != ref.labels).sum())} labels differ"
        assert np.array_equal(sp["n"], ref.sp["n"]) and np.array_equal(sp["sum_x"], ref.sp["sum_x"]), env
        outs.append(info.counters().copy())
    for c in outs[1:]:
        assert np.array_equal(c, outs[0]), "per-phase counters differ between variants"


def test_graph_replay_follows_inputs_and_params():
    import torch
    w = synth.scaled(3, 512, 512)
    img1 = w.images()
    w2 = synth.scaled(3, 512, 512, seed_offset=7)
    img2 = w2.images()
    r = make_ctx({}, w.pixels, w.params.n_superpixels)
    try:
        t = torch.from_numpy(img1).cuda()
        labels = torch.empty((1, w.H, w.W), dtype=torch.int32, device="cuda")
        r.segment(t, w.params, labels)  # capture
        r.segment(t, w.params, labels)  # replay
        torch.cuda.synchronize()
        assert np.array_equal(labels.cpu().numpy(), oracle.segment(img1, w.params).labels)
        t.copy_(torch.from_numpy(img2))  # same buffer, new contents: the replay must see them
        r.segment(t, w.params, labels)
        torch.cuda.synchronize()
        assert np.array_equal(labels.cpu().numpy(), oracle.segment(img2, w.params).labels)
        p2 = copy.deepcopy(w.params)  # new params: a new graph
        p2.sweeps = 2
        p2.size_mode = synth.SIZE_HARD
        r.segment(t, p2, labels)
        torch.cuda.synchronize()
        assert np.array_equal(labels.cpu().numpy(), oracle.segment(img2, p2).labels)
    finally:
        r.close()


@pytest.mark.parametrize("setting", synth.SETTINGS)
def test_comparison_settings_oracle_exact(setting):
    """CTFTPS (HARD, no mask), multi-scale CTFTPS (+ RECOUNT) and RAPID (MERGE +
    CLASS + REUSE) on a 768^2 sample with config 4's densities, bit-exact with the oracle."""
    w = synth.with_setting(synth.scaled(4, 768, 768), setting)
    img = w.images()
    ref = oracle.segment(img, w.params)
    r = make_ctx({}, w.pixels, w.params.n_superpixels)
    try:
        lab, sp, info = gpu_run(r, img, w.params)
    finally:
        r.close()
    assert np.array_equal(lab, ref.labels)
    assert np.array_equal(sp["n"], ref.sp["n"])
    assert info.status == 0
    assert np.array_equal(info.counters()[..., oracle.C_COMMIT], ref.counters[..., oracle.C_COMMIT])


@pytest.mark.parametrize("stats_mode", [0, 1])
def test_host_stream_api_pipelined_oracle_exact(stats_mode):
    """rapid_segment_host_stream: n host images through two device buffer pairs and two copy
    streams; every output equals the oracle (also with RECOUNT integrity checks on)."""
    import torch
    n = 5
    ws = [synth.scaled(3, 384, 384, seed_offset=k) for k in range(n)]
    for w in ws:
        w.params.stats_mode = stats_mode
    imgs = []
    for w in ws:
        h = torch.empty((1, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
        w.images(out=h.numpy())
        imgs.append(h.numpy())
    labs = [torch.empty((1, ws[0].H, ws[0].W), dtype=torch.int32).pin_memory().numpy() for _ in range(n)]
    r = make_ctx({}, ws[0].pixels, ws[0].params.n_superpixels)
    try:
        r.segment_host_stream(imgs, ws[0].params, labs)
    finally:
        r.close()
    for k in range(n):
        ref = oracle.segment(imgs[k], ws[0].params)
        assert np.array_equal(labs[k], ref.labels), f"image {k}"


@pytest.mark.parametrize("cfg,side,eps", [(1, 0, 0), (1, 0, 2), (3, 512, 2), (5, 0, 1)])
def test_quality_metrics_match_oracle(cfg, side, eps):
    """f4: UE and BR of the GPU segmentation against the generator's ground-truth
    segments, computed by rapid_quality on the GPU, equal the oracle's exact counts."""
    import torch
    w = synth.scaled(cfg, side, side) if side else synth.config(cfg)
    if cfg == 5:
        w.seeds, w.regions, w.nuclei, w.B = w.seeds[:3], w.regions[:3], w.nuclei[:3], 3
    img, gt = w.images(), w.segments()
    r = make_ctx({}, w.pixels, w.B * w.params.n_superpixels)
    try:
        lab = r.segment(torch.from_numpy(img).cuda(), w.params)
        q = r.quality(lab, torch.from_numpy(gt).cuda(), w.params.n_superpixels, eps)
        ref = oracle.quality(lab.cpu().numpy(), gt, eps)
    finally:
        r.close()
    for k in ("pixels", "leak", "gt_boundary", "covered"):
        assert q[k] == ref[k], k
    assert 0.0 <= q["ue"] < 1.0 and 0.0 < q["br"] <= 1.0


def test_quality_closed_forms_on_gpu():
    import torch
    g = np.zeros((1, 8, 8), np.int32)
    g[..., 4:] = 1
    lab = np.zeros((1, 8, 8), np.int32)
    lab[..., 5:] = 1
    r = make_ctx({}, 64, 4)
    try:
        q0 = r.quality(torch.from_numpy(lab).cuda(), torch.from_numpy(g).cuda(), 2, 0)
        q1 = r.quality(torch.from_numpy(lab).cuda(), torch.from_numpy(g).cuda(), 2, 1)
        qi = r.quality(torch.from_numpy(g).cuda(), torch.from_numpy(g).cuda(), 2, 0)
    finally:
        r.close()
    assert q0["ue"] == 0.25 and q0["br"] == 0.5 and q1["br"] == 1.0
    assert qi["ue"] == 0.0 and qi["br"] == 1.0


@pytest.mark.parametrize("cfg,side,mask", [(3, 512, 1), (3, 384, 2), (4, 512, 3), (5, 0, 1)])
def test_feature_model_prediction_oracle_exact(cfg, side, mask):
    """f2 (A31): prediction by the linear model on the 4 superpixel features — labels,
    y and active flags bit-exact with the oracle, for every mask rule that uses y."""
    w = synth.scaled(cfg, side, side) if side else synth.config(cfg)
    if cfg == 5:
        w.seeds, w.regions, w.nuclei, w.B = w.seeds[:3], w.regions[:3], w.nuclei[:3], 3
    p = copy.deepcopy(w.params)
    p.y_model, p.mask_rule = synth.Y_FEATURES, mask
    p.feat_w_q16 = [round(0.6 * 65536), -65536, 20000, -90000, 30000]  # every feature matters
    img = w.images()
    ref = oracle.segment(img, p)
    r = make_ctx({}, w.pixels, w.B * p.n_superpixels)
    try:
        lab, sp, info = gpu_run(r, img, p)
    finally:
        r.close()
    assert np.array_equal(sp["y"], ref.sp["y"]), f"y differs at {int((sp['y'] != ref.sp['y']).sum())} superpixels"
    alive = ref.sp["alive"] == 1
    assert np.array_equal(sp["active"][alive], ref.sp["active"][alive])
    assert np.array_equal(lab, ref.labels)


@pytest.mark.parametrize("cfg,side", [(1, 0), (2, 0), (3, 512), (5, 0)])
def test_literal_pyramid_mode_oracle_exact(cfg, side):
    """f3 (Eq. 8 with the paper's approximation; A32): block colour data from rounded
    box-mean levels, S_1 from the coarsest level — bit-exact with the oracle (labels, sums,
    counters), including the non-dyadic geometry of config 1."""
    w = synth.scaled(cfg, side, side) if side else synth.config(cfg)
    if cfg == 5:
        w.seeds, w.regions, w.nuclei, w.B = w.seeds[:3], w.regions[:3], w.nuclei[:3], 3
    p = copy.deepcopy(w.params)
    p.stats_mode = synth.STATS_PYRAMID
    img = w.images()
    ref = oracle.segment(img, p)
    r = make_ctx({}, w.pixels, w.B * p.n_superpixels)
    try:
        lab, sp, info = gpu_run(r, img, p)
    finally:
        r.close()
    assert np.array_equal(lab, ref.labels)
    for f in ("n", "sum_r", "sum_g", "sum_b", "sum_x", "sum_y"):
        assert np.array_equal(sp[f], ref.sp[f]), f
    assert np.array_equal(info.counters()[..., oracle.C_COMMIT], ref.counters[..., oracle.C_COMMIT])


def test_random_cases_through_64bit_block_variant():
    """The randomized all-options sweep again with every block stage forced onto K4's 64-bit
    position-factor variant (RAPID_SWEEP_NO_SMALLB=1): bit-exact with the oracle."""
    from test_gpu_parity import random_all_options
    r = make_ctx({"RAPID_SWEEP_NO_SMALLB": "1"}, 1 << 22, 1 << 16)
    try:
        random_all_options(r, 77, 16)
    finally:
        r.close()


def test_random_cases_through_candidate_list():
    """The randomized all-options sweep with every block stage (b >= 2) evaluated from the
    per-phase candidate list (RAPID_SWEEP_LIST=2: k_bset_list + k_sweep<LIST>), once with the
    64-bit position-factor variant too: bit-exact with the oracle."""
    from test_gpu_parity import random_all_options
    for env, seed in (({"RAPID_SWEEP_LIST": "2"}, 53), ({"RAPID_SWEEP_LIST": "2", "RAPID_SWEEP_NO_SMALLB": "1"}, 54)):
        r = make_ctx(env, 1 << 22, 1 << 16)
        try:
            random_all_options(r, seed, 12)
        finally:
            r.close()


@pytest.mark.parametrize("lim", [60, 150, 600])
def test_random_cases_packed_delta_switch(lim):
    """K5 packs its stats deltas (3 REDs per run, folded by K3) only while every snapshot size
    is within the stage's limit; RAPID_PACKED_LIM caps that limit near the random cases'
    superpixel sizes so that calls run packed, direct, or switch to direct once merges grow a
    superpixel past it: bit-exact with the oracle in every case.  (Calls this small take the
    direct REDs by default; RAPID_PACKED=1 forces the packed path.)"""
    from test_gpu_parity import random_all_options
    r = make_ctx({"RAPID_PACKED": "1", "RAPID_PACKED_LIM": str(lim)}, 1 << 22, 1 << 16)
    try:
        random_all_options(r, 91 + lim, 12)
    finally:
        r.close()


def test_host_stream_long_run_drains_flag_ring():
    """rapid_segment_host_stream over n = 70 > 64 images with RECOUNT integrity checks: the
    pinned 64-entry error-flag ring is drained once mid-stream and the 6-entry tail at the end;
    every output equals the oracle and the call reports no integrity failure."""
    import torch
    n = 70
    ws = [synth.scaled(3, 64, 64, seed_offset=k) for k in range(n)]
    p = copy.deepcopy(ws[0].params)
    p.stats_mode = synth.STATS_RECOUNT
    imgs, labs = [], []
    for w in ws:
        h = torch.empty((1, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
        w.images(out=h.numpy())
        imgs.append(h.numpy())
        labs.append(torch.empty((1, w.H, w.W), dtype=torch.int32).pin_memory().numpy())
    r = make_ctx({}, ws[0].pixels, p.n_superpixels)
    try:
        r.segment_host_stream(imgs, p, labs)  # raises RapidError on an integrity failure
    finally:
        r.close()
    for k in range(n):
        assert np.array_equal(labs[k], oracle.segment(imgs[k], p).labels), f"image {k}"


def test_random_cases_through_row_walking_bset_pass():
    """The row-walking parent-map boundary-set pass runs only on stages with >= 32768 tiles by
    default (configs 3 and 4); forced everywhere (RAPID_BSET_ROWS=2) the randomized all-options
    sweep — ragged tiles, batches, every mask rule — stays bit-exact with the oracle."""
    from test_gpu_parity import random_all_options
    r = make_ctx({"RAPID_BSET_ROWS": "2"}, 1 << 22, 1 << 16)
    try:
        random_all_options(r, 79, 24)
    finally:
        r.close()


def test_host_stream_batches():
    """rapid_segment_host_stream with batches (B = 3 images per segmentation call, 4 calls):
    every image of every call equals the oracle's."""
    import torch
    w = synth.scaled(5, 256, 256, B=3)
    imgs, labs, refs = [], [], []
    for k in range(4):
        wk = synth.scaled(5, 256, 256, B=3, seed_offset=10 * k)
        h = torch.empty((3, 256, 256, 3), dtype=torch.uint8).pin_memory()
        wk.images(out=h.numpy())
        imgs.append(h.numpy())
        labs.append(torch.empty((3, 256, 256), dtype=torch.int32).pin_memory().numpy())
        refs.append(oracle.segment(imgs[-1], w.params).labels)
    r = make_ctx({}, w.pixels, w.B * w.params.n_superpixels)
    try:
        r.segment_host_stream(imgs, w.params, labs)
    finally:
        r.close()
    for k in range(4):
        assert np.array_equal(labs[k], refs[k]), f"call {k}"


def test_profiling_levels_time_the_same_segmentation():
    """rapid_set_profiling levels 1 (events around every launch group), 2 (+ window counting) and
    3 (coarse: each stage's phase loop as one interval, no events between K3/K4/K5) change only
    what is timed: labels and counters are those of level 0, level 3 reports no K3/K4/K5 class
    and a phase-set interval per stage that ran, and it is not longer than level 1's interval
    with its inner events by more than noise."""
    import torch
    import paper_1704_02083_b200 as rb
    w = synth.scaled(4, 1024, 1024)
    img = torch.from_numpy(w.images()).cuda()
    r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=w.params.n_superpixels)
    try:
        base = r.segment(img, w.params).cpu().numpy()
        _, info0 = r.stats(0)
        c0 = info0.counters()
        ms = {}
        for level in (1, 2, 3):
            r.set_profiling(level)
            r.segment(img, w.params)                  # capture at this level
            best = None
            for _ in range(5):
                lab = r.segment(img, w.params)        # replay
                m = r.profile().ms_array()
                best = m if best is None else np.minimum(best, m)
            assert np.array_equal(lab.cpu().numpy(), base), level
            _, info = r.stats(0)
            assert np.array_equal(info.counters(), c0), level
            ms[level] = best
        nst = len(w.params.block_sizes)
        assert (ms[3][rb.K_PHASESET][:nst] > 0).all()
        for k in (rb.K_SNAPSHOT, rb.K_PROPOSE, rb.K_COMMIT, rb.K_EVAL):
            assert ms[3][k].sum() == 0, k
            assert k == rb.K_EVAL or ms[1][k].sum() > 0, k
        for k in (rb.K_PYRAMID, rb.K_MERGE, rb.K_TRANSITION, rb.K_FINAL):
            assert ms[3][k].sum() > 0, k
        assert ms[3][rb.K_PHASESET].sum() <= 1.05 * ms[1][rb.K_PHASESET].sum()
        r.set_profiling(0)
        assert np.array_equal(r.segment(img, w.params).cpu().numpy(), base)
    finally:
        r.close()

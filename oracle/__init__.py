"""ctypes binding of the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this package.  The product path
(paper_1704_02083_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
MAX_STAGES = 12
MAX_SWEEPS = 64
NCNT = 6
C_CAND, C_TOPO, C_PROP, C_SIZEREJ, C_COMMIT, C_COMMREJ = range(6)
STOP_NONE, STOP_PHASE, STOP_STAGE_START, STOP_AFTER_MERGE, STOP_AFTER_PREDICT = range(5)


class OrcQuality(ctypes.Structure):
    _fields_ = [("pixels", ctypes.c_int64), ("leak", ctypes.c_int64), ("gt_boundary", ctypes.c_int64),
                ("covered", ctypes.c_int64)]


def quality(labels, gt, eps=2):
    """f4: under-segmentation error and boundary recall of labels [B][H][W] against the
    ground-truth segment map gt (same shape).  Returns dict(ue, br, pixels, leak, gt_boundary,
    covered); br = 1.0 when gt has no boundary pixel."""
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    g = np.ascontiguousarray(gt, dtype=np.int32)
    if lab.ndim == 2:
        lab, g = lab[None], g[None]
    assert lab.shape == g.shape
    B, H, W = lab.shape
    q = OrcQuality()
    rc = lib().orc_quality_eval(lab.ctypes.data, g.ctypes.data, B, H, W, int(eps), ctypes.byref(q))
    if rc:
        raise ValueError(f"orc_quality_eval failed ({rc})")
    return {"ue": q.leak / q.pixels, "br": (q.covered / q.gt_boundary) if q.gt_boundary else 1.0,
            "pixels": q.pixels, "leak": q.leak, "gt_boundary": q.gt_boundary, "covered": q.covered}


class OrcParams(ctypes.Structure):
    _fields_ = [
        ("n_superpixels", ctypes.c_int32),
        ("n_stages", ctypes.c_int32),
        ("block_size", ctypes.c_int32 * MAX_STAGES),
        ("sweeps", ctypes.c_int32),
        ("lambda_pos_q16", ctypes.c_int64),
        ("lambda_b_q16", ctypes.c_int64),
        ("size_mode", ctypes.c_int32),
        ("l_num", ctypes.c_int32),
        ("l_den", ctypes.c_int32),
        ("u_num", ctypes.c_int32),
        ("u_den", ctypes.c_int32),
        ("mask_rule", ctypes.c_int32),
        ("n_proto", ctypes.c_int32),
        ("proto", (ctypes.c_int32 * 3) * 4),
        ("tau2", ctypes.c_int64),
        ("stats_mode", ctypes.c_int32),
        ("y_model", ctypes.c_int32),
        ("feat_w_q16", ctypes.c_int64 * 5),
    ]


SP_DTYPE = np.dtype([
    ("n", "<i8"), ("sum_r", "<i8"), ("sum_g", "<i8"), ("sum_b", "<i8"),
    ("sum_x", "<i8"), ("sum_y", "<i8"), ("init_size", "<i4"),
    ("alive", "i1"), ("active", "i1"), ("y", "i1"), ("pad", "i1"),
], align=True)

MOVE_DTYPE = np.dtype([
    ("stage", "<i4"), ("sweep", "<i4"), ("phase", "<i4"), ("img", "<i4"),
    ("bi", "<i4"), ("bj", "<i4"), ("A", "<i4"), ("B", "<i4"),
    ("dE_hi", "<i8"), ("dE_lo", "<u8"),
], align=True)

MERGE_DTYPE = np.dtype([
    ("stage", "<i4"), ("img", "<i4"), ("A", "<i4"), ("T", "<i4"),
    ("len", "<i8"), ("dE_hi", "<i8"), ("dE_lo", "<u8"),
], align=True)


class OrcDebug(ctypes.Structure):
    _fields_ = [
        ("stop_kind", ctypes.c_int32),
        ("stop_stage", ctypes.c_int32),
        ("stop_sweep", ctypes.c_int32),
        ("stop_phase", ctypes.c_int32),
        ("map_out", ctypes.c_void_p),
        ("map_cap", ctypes.c_int64),
        ("map_nbx", ctypes.c_int32),
        ("map_nby", ctypes.c_int32),
        ("stopped", ctypes.c_int32),
        ("moves", ctypes.c_void_p),
        ("moves_cap", ctypes.c_int64),
        ("n_moves", ctypes.c_int64),
        ("merges", ctypes.c_void_p),
        ("merges_cap", ctypes.c_int64),
        ("n_merges", ctypes.c_int64),
        ("phase_counters", ctypes.c_void_p),
        ("stage_victims", ctypes.c_int64 * MAX_STAGES),
        ("stage_merges", ctypes.c_int64 * MAX_STAGES),
        ("victim_out", ctypes.c_void_p),
    ]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        # RAPID_ORACLE_LIB: a mutated build for the mutation check (tests/mutation_check.sh)
        path = os.environ.get("RAPID_ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle`")
        L = ctypes.CDLL(path)
        L.orc_segment.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(OrcParams), ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.POINTER(OrcDebug)]
        L.orc_segment.restype = ctypes.c_int
        L.orc_grid.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.orc_grid.restype = ctypes.c_int
        L.orc_stage_axis.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_int]
        L.orc_stage_axis.restype = ctypes.c_int
        L.orc_yokoi_c4.argtypes = [ctypes.c_int]
        L.orc_yokoi_c4.restype = ctypes.c_int
        L.orc_round_mean.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.orc_round_mean.restype = None
        L.orc_colour_mean.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.orc_colour_mean.restype = None
        L.orc_block_move.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.POINTER(OrcParams), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_uint64)]
        L.orc_block_move.restype = ctypes.c_int
        L.orc_quality_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(OrcQuality)]
        L.orc_quality_eval.restype = ctypes.c_int
        _LIB = L
    return _LIB


def make_params(p) -> OrcParams:
    """p: synth.Params (or any object with the same fields)."""
    o = OrcParams()
    o.n_superpixels = p.n_superpixels
    o.n_stages = len(p.block_sizes)
    for i, b in enumerate(p.block_sizes):
        o.block_size[i] = b
    o.sweeps = p.sweeps
    o.lambda_pos_q16 = p.lambda_pos_q16
    o.lambda_b_q16 = p.lambda_b_q16
    o.size_mode = p.size_mode
    o.l_num, o.l_den, o.u_num, o.u_den = p.l_num, p.l_den, p.u_num, p.u_den
    o.mask_rule = p.mask_rule
    o.n_proto = len(p.protos)
    for k, pr in enumerate(p.protos):
        for ch in range(3):
            o.proto[k][ch] = pr[ch]
    o.tau2 = p.tau2
    o.stats_mode = p.stats_mode
    o.y_model = getattr(p, "y_model", 0)
    for i, v in enumerate(getattr(p, "feat_w_q16", [0] * 5)):
        o.feat_w_q16[i] = v
    return o


class Result:
    def __init__(self, labels, sp, dbg, moves, merges, counters, map_out):
        self.labels = labels
        self.sp = sp
        self.dbg = dbg
        self.moves = moves
        self.merges = merges
        self.counters = counters
        self.map = map_out

    @property
    def stage_victims(self):
        return list(self.dbg.stage_victims)

    @property
    def stage_merges(self):
        return list(self.dbg.stage_merges)


def i128(hi, lo):
    return (int(hi) << 64) | int(lo)


def segment(image, params, stop=None, log_moves=0, log_merges=0, map_cap=0):
    """Run the oracle. image: u8 [B][H][W][3] (or [H][W][3]); params: synth.Params.
    stop: None or (kind, stage, sweep, phase).  Returns Result."""
    img = np.ascontiguousarray(image, dtype=np.uint8)
    if img.ndim == 3:
        img = img[None]
    B, H, W, _ = img.shape
    M = params.n_superpixels
    labels = np.full((B, H, W), -1, dtype=np.int32)
    sp = np.zeros(B * M, dtype=SP_DTYPE)
    op = make_params(params)
    dbg = OrcDebug()
    counters = np.zeros((MAX_STAGES, MAX_SWEEPS, 4, NCNT), dtype=np.int64)
    dbg.phase_counters = counters.ctypes.data
    moves = np.zeros(max(log_moves, 0), dtype=MOVE_DTYPE)
    merges = np.zeros(max(log_merges, 0), dtype=MERGE_DTYPE)
    if log_moves:
        dbg.moves = moves.ctypes.data
        dbg.moves_cap = log_moves
    if log_merges:
        dbg.merges = merges.ctypes.data
        dbg.merges_cap = log_merges
    map_out = None
    victims = np.zeros(B * M, dtype=np.uint8)
    if stop is not None:
        dbg.victim_out = victims.ctypes.data
        dbg.stop_kind, dbg.stop_stage, dbg.stop_sweep, dbg.stop_phase = stop
        cap = map_cap or B * (H + 2) * (W + 2) * 2
        map_out = np.full(cap, -7, dtype=np.int32)
        dbg.map_out = map_out.ctypes.data
        dbg.map_cap = cap
    rc = lib().orc_segment(img.ctypes.data, B, H, W, ctypes.byref(op), labels.ctypes.data,
                           sp.ctypes.data, ctypes.byref(dbg))
    if rc != 0:
        raise OracleError(rc)
    if map_out is not None and dbg.stopped:
        map_out = map_out[: B * dbg.map_nby * dbg.map_nbx].reshape(B, dbg.map_nby, dbg.map_nbx)
    res = Result(labels, sp, dbg, moves[: dbg.n_moves], merges[: dbg.n_merges], counters, map_out)
    res.victims = victims if (stop is not None and dbg.stopped) else None
    return res


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle returned {rc}")
        self.rc = rc


def grid(H, W, M):
    r, c = ctypes.c_int(), ctypes.c_int()
    rc = lib().orc_grid(H, W, M, ctypes.byref(r), ctypes.byref(c))
    if rc:
        raise OracleError(rc)
    return r.value, c.value


def stage_axis(length, b, cuts):
    cuts = np.ascontiguousarray(cuts, dtype=np.int32)
    cap = length // b + len(cuts) + 3
    out = np.zeros(cap, dtype=np.int32)
    n = lib().orc_stage_axis(length, b, cuts.ctypes.data, len(cuts), out.ctypes.data, cap)
    if n < 0:
        raise OracleError(n)
    return out[:n]


def yokoi_c4(mask):
    return lib().orc_yokoi_c4(mask)


def block_move(win, means, d, e, params):
    """One block's decision (O6 steps 2-6, no gates). win: 9 labels row-major (-1 outside);
    means: [9][5] (cq r,g,b, mq x,y) of each cell's label; d: [6] block data; e: [4] edges
    N,E,S,W.  Returns (code, B, dE): code 0 not boundary, 1 not simple, 2 no move, 3 move."""
    w = np.ascontiguousarray(win, dtype=np.int32)
    m = np.ascontiguousarray(means, dtype=np.int64)
    dd = np.ascontiguousarray(d, dtype=np.int64)
    ee = np.ascontiguousarray(e, dtype=np.int64)
    B, hi, lo = ctypes.c_int32(-1), ctypes.c_int64(0), ctypes.c_uint64(0)
    op = make_params(params)
    code = lib().orc_block_move(w.ctypes.data, m.ctypes.data, dd.ctypes.data, ee.ctypes.data,
                                ctypes.byref(op), ctypes.byref(B), ctypes.byref(hi), ctypes.byref(lo))
    return code, B.value, i128(hi.value, lo.value) if code == 3 else None


def round_mean(S, n):
    q = ctypes.c_int64()
    lib().orc_round_mean(S, n, ctypes.byref(q))
    return q.value


def colour_mean(S, n):
    """O5's rounding of a colour channel's mean, clamped to [0, 255] (DESIGN A33)."""
    q = ctypes.c_int64()
    lib().orc_colour_mean(S, n, ctypes.byref(q))
    return q.value

"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NO arithmetic of the RAPID method (no grid, energy, means or
moves): it only produces images (via the C generator ``synth.c``) and the five
workload configurations of BASELINE.json ``configs`` with their method
parameters stored as plain integers.  See DESIGN.md §3 for the recipe.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, asdict

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _SynthParams(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("H", ctypes.c_int32),
        ("W", ctypes.c_int32),
        ("n_regions", ctypes.c_int32),
        ("n_nuclei", ctypes.c_int32),
        ("bg_permille", ctypes.c_int32),
        ("noise_sigma", ctypes.c_int32),
    ]


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} synth`")
        lib = ctypes.CDLL(path)
        lib.synth_image.argtypes = [ctypes.POINTER(_SynthParams), ctypes.c_void_p, ctypes.c_int]
        lib.synth_image.restype = ctypes.c_int
        lib.synth_segments.argtypes = [ctypes.POINTER(_SynthParams), ctypes.c_void_p, ctypes.c_int]
        lib.synth_segments.restype = ctypes.c_int
        lib.synth_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        lib.synth_hash.restype = ctypes.c_uint64
        _LIB = lib
    return _LIB


def image(H, W, seed, n_regions, n_nuclei, bg_permille=0, noise_sigma=8, nthreads=0, out=None):
    """Return a u8 [H][W][3] synthetic H&E-like image (numpy)."""
    if out is None:
        out = np.empty((H, W, 3), dtype=np.uint8)
    assert out.dtype == np.uint8 and out.shape == (H, W, 3) and out.flags.c_contiguous
    p = _SynthParams(seed, H, W, n_regions, n_nuclei, bg_permille, noise_sigma)
    rc = _lib().synth_image(ctypes.byref(p), out.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError(f"synth_image failed ({rc})")
    return out


def segments(H, W, seed, n_regions, n_nuclei, bg_permille=0, nthreads=0, out=None):
    """Ground-truth segment map int32 [H][W] of the same generator parameters: tissue region k,
    background cell n_regions + j, or nucleus n_regions + 64 + k (the blob painted last)."""
    if out is None:
        out = np.empty((H, W), dtype=np.int32)
    assert out.dtype == np.int32 and out.shape == (H, W) and out.flags.c_contiguous
    p = _SynthParams(seed, H, W, n_regions, n_nuclei, bg_permille, 0)
    rc = _lib().synth_segments(ctypes.byref(p), out.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError(f"synth_segments failed ({rc})")
    return out


def hash3(seed, stream, index):
    return int(_lib().synth_hash(seed, stream, index))


# --------------------------------------------------------------------------
# Method parameters (integers only).  Field meanings follow include/rapid.h;
# the oracle has its own struct with the same field meanings.
SIZE_NONE, SIZE_HARD, SIZE_MERGE = 0, 1, 2
MASK_OFF, MASK_CLASS, MASK_BSP, MASK_EQ7 = 0, 1, 2, 3
STATS_REUSE, STATS_RECOUNT, STATS_PYRAMID = 0, 1, 2
Y_PROTO, Y_FEATURES = 0, 1
# SURVEY f2 default linear model (training is out of scope; a hand-set model file): tissue
# (pink / purple) is darker than the white background, y = +1 iff 0.85 - f1 >= 0, i.e. mean
# brightness <= 0.85 * 255.  Bias, w1..w4 in Q16.16.
FEAT_W_TISSUE = (round(0.85 * 65536), -65536, 0, 0, 0)

PROTO_PINK = (230, 170, 200)
PROTO_PURPLE = (120, 70, 150)
# tau^2 in intensity^2 units, calibrated once on config 3 (DESIGN.md §3 "tau");
# y=+1 iff min_k ||c - proto_k||^2 <= TAU2.
TAU2 = 1600


def lambda_pos_default(H, W, M):
    """SLIC-like lambda_pos = 400 / InitSize_mean in Q16, rounded half up."""
    return (2 * 400 * 65536 * M + H * W) // (2 * H * W)


LAMBDA_B_DEFAULT = 32 * 65536


@dataclass
class Params:
    n_superpixels: int
    block_sizes: list
    sweeps: int = 5
    lambda_pos_q16: int = 0
    lambda_b_q16: int = LAMBDA_B_DEFAULT
    size_mode: int = SIZE_NONE
    l_num: int = 1
    l_den: int = 4
    u_num: int = 3
    u_den: int = 2
    mask_rule: int = MASK_OFF
    protos: list = field(default_factory=lambda: [PROTO_PINK, PROTO_PURPLE])
    tau2: int = TAU2
    stats_mode: int = STATS_REUSE
    y_model: int = Y_PROTO
    feat_w_q16: list = field(default_factory=lambda: list(FEAT_W_TISSUE))

    def asdict(self):
        return asdict(self)


@dataclass
class Workload:
    name: str
    B: int
    H: int
    W: int
    seeds: list
    regions: list
    nuclei: list
    bg_permille: int
    params: Params

    @property
    def pixels(self):
        return self.B * self.H * self.W

    def segments(self, nthreads=0, out=None):
        """Ground-truth segment maps int32 [B][H][W] (per-image ids, see segments())."""
        if out is None:
            out = np.empty((self.B, self.H, self.W), dtype=np.int32)
        for b in range(self.B):
            segments(self.H, self.W, self.seeds[b], self.regions[b], self.nuclei[b], self.bg_permille, nthreads,
                     out=out[b])
        return out

    def images(self, nthreads=0, out=None):
        if out is None:
            out = np.empty((self.B, self.H, self.W, 3), dtype=np.uint8)
        for b in range(self.B):
            image(self.H, self.W, self.seeds[b], self.regions[b], self.nuclei[b],
                  self.bg_permille, 8, nthreads, out=out[b])
        return out


def config(k: int) -> Workload:
    """BASELINE.json configs[k-1] (k = 1..5) as a Workload."""
    if k == 1:
        H, W, M = 321, 481, 400
        return Workload("cfg1_481x321", 1, H, W, [1], [12], [40], 0,
                        Params(M, [16, 8, 4, 2, 1], 5, lambda_pos_default(H, W, M)))
    if k == 2:
        H = W = 2048
        M = 4096
        return Workload("cfg2_2048", 1, H, W, [2], [300], [4000], 0,
                        Params(M, [32, 16, 8, 4, 2, 1], 5, lambda_pos_default(H, W, M),
                               size_mode=SIZE_MERGE))
    if k == 3:
        H = W = 8192
        M = 65536
        return Workload("cfg3_8192", 1, H, W, [3], [5000], [60000], 200,
                        Params(M, [32, 16, 8, 4, 2, 1], 5, lambda_pos_default(H, W, M),
                               size_mode=SIZE_MERGE, mask_rule=MASK_CLASS))
    if k == 4:
        H = W = 32768
        M = 1 << 20
        return Workload("cfg4_32768", 1, H, W, [4], [80000], [1000000], 600,
                        Params(M, [32, 16, 8, 4, 2, 1], 5, lambda_pos_default(H, W, M),
                               size_mode=SIZE_MERGE, mask_rule=MASK_CLASS))
    if k == 5:
        H = W = 1024
        M = 1024
        seeds = list(range(100, 164))
        regions = [50 + hash3(s, 7, 0) % 451 for s in seeds]
        return Workload("cfg5_64x1024", 64, H, W, seeds, regions, [1000] * 64, 200,
                        Params(M, [32, 16, 8, 4, 2, 1], 5, lambda_pos_default(H, W, M),
                               size_mode=SIZE_MERGE, mask_rule=MASK_CLASS))
    raise ValueError(k)


def scaled(k: int, H: int, W: int, B: int = 1, seed_offset: int = 0) -> Workload:
    """A smaller workload with config k's densities (regions, nuclei, superpixels per pixel)
    and parameters; used for bounded CPU samples and mid-size parity cases."""
    base = config(k)
    frac = (H * W) / (base.H * base.W)
    M = max(1, round(base.params.n_superpixels * frac))
    p = Params(**base.params.asdict())
    p.n_superpixels = M
    p.lambda_pos_q16 = lambda_pos_default(H, W, M)
    seeds = [base.seeds[0] + 1000 + seed_offset + b for b in range(B)]
    regions = [max(1, round(base.regions[0] * frac))] * B
    nuclei = [round(base.nuclei[0] * frac)] * B
    return Workload(f"{base.name}_sample{H}x{W}x{B}", B, H, W, seeds, regions, nuclei,
                    base.bg_permille, p)


# the paper's comparison settings on this path (Table 1).  They
# only configure the existing kernels (run_ctftps / run_multiscale / run_rapid).
SETTINGS = ("rapid", "ctftps", "multiscale", "rapid_features", "rapid_pyramid")


def with_setting(w: Workload, setting: str) -> Workload:
    """Copy of workload `w` under one of SETTINGS: RAPID = the config's own parameters;
    rapid_features = RAPID with the f2 feature-model prediction (FEAT_W_TISSUE);
    rapid_pyramid = RAPID on the f3 literal image pyramid (STATS_PYRAMID);
    CTFTPS = HARD size bound, no mask, REUSE; multi-scale CTFTPS = the same with statistics
    recounted at every stage (RECOUNT)."""
    import copy
    if setting not in SETTINGS:
        raise ValueError(setting)
    w2 = copy.deepcopy(w)
    if setting == "rapid":  # the config's own parameters (configs 3-5: MERGE + CLASS + REUSE)
        return w2
    p = w2.params
    if setting == "rapid_pyramid":  # f3: RAPID on a literal image pyramid (approximate Eq. 8)
        p.size_mode, p.mask_rule, p.stats_mode = SIZE_MERGE, MASK_CLASS, STATS_PYRAMID
        w2.name = f"{w.name}_{setting}"
        return w2
    if setting == "rapid_features":  # f2: the prediction by the feature model (tissue model)
        p.size_mode, p.mask_rule, p.stats_mode = SIZE_MERGE, MASK_CLASS, STATS_REUSE
        p.y_model, p.feat_w_q16 = Y_FEATURES, list(FEAT_W_TISSUE)
        w2.name = f"{w.name}_{setting}"
        return w2
    p.size_mode, p.mask_rule = SIZE_HARD, MASK_OFF
    p.stats_mode = STATS_RECOUNT if setting == "multiscale" else STATS_REUSE
    w2.name = f"{w.name}_{setting}"
    return w2


"""paper_1704_02083_b200 — B200-native RAPID / CTFTPS superpixel refinement.

Thin ctypes binding over the C ABI in include/rapid.h (librapid.so, built in-tree by
``make lib`` / ``__graft_entry__.build()``).  Argument marshalling only: every step of the
method runs in the sm_100a kernels.  PyTorch supplies device memory and the stream.
There is no CPU fallback: importing this package without librapid.so raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAPID_LIB", os.path.join(_HERE, "librapid.so"))  # override: A/B builds

MAX_STAGES = 12
MAX_SWEEPS = 64
MAX_PROTO = 4
NCNT = 6
NK = 10
C_CAND, C_TOPO, C_PROP, C_SIZEREJ, C_COMMIT, C_COMMREJ = range(6)
(K_PYRAMID, K_SNAPSHOT, K_PROPOSE, K_COMMIT, K_MERGE, K_PREDICT, K_TRANSITION, K_FINAL, K_PHASESET,
 K_EVAL) = range(10)  # K_PROPOSE = K4a scan (the HBM-streaming kernel), K_EVAL = K4b
STOP_NONE, STOP_PHASE, STOP_STAGE_START, STOP_AFTER_MERGE, STOP_AFTER_PREDICT = range(5)
STATUS = {0: "ok", -1: "E_ARG", -2: "E_CAPACITY", -3: "E_RANGE", -4: "E_CUDA", -5: "E_OOM",
          -6: "E_INTEGRITY", -7: "E_STATE"}


class rapid_params(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("batch", ctypes.c_uint32),
        ("n_superpixels", ctypes.c_uint32),
        ("n_stages", ctypes.c_uint32),
        ("block_size", ctypes.c_uint32 * MAX_STAGES),
        ("sweeps", ctypes.c_uint32),
        ("pad0_", ctypes.c_uint8 * 4),
        ("lambda_pos_q16", ctypes.c_int64),
        ("lambda_b_q16", ctypes.c_int64),
        ("size_mode", ctypes.c_uint32),
        ("l_num", ctypes.c_uint32),
        ("l_den", ctypes.c_uint32),
        ("u_num", ctypes.c_uint32),
        ("u_den", ctypes.c_uint32),
        ("mask_rule", ctypes.c_uint32),
        ("n_proto", ctypes.c_uint32),
        ("proto_rgb", (ctypes.c_uint8 * 3) * MAX_PROTO),
        ("pad_", ctypes.c_uint8 * 8),
        ("tau2", ctypes.c_int64),
        ("stats_mode", ctypes.c_uint32),
        ("y_model", ctypes.c_uint32),
        ("feat_w_q16", ctypes.c_int64 * 5),
    ]


class rapid_sp_stat(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("sum_r", ctypes.c_int64), ("sum_g", ctypes.c_int64),
        ("sum_b", ctypes.c_int64), ("sum_x", ctypes.c_int64), ("sum_y", ctypes.c_int64),
        ("mean_r", ctypes.c_double), ("mean_g", ctypes.c_double), ("mean_b", ctypes.c_double),
        ("mean_x", ctypes.c_double), ("mean_y", ctypes.c_double),
        ("init_size", ctypes.c_int32),
        ("alive", ctypes.c_int8), ("active", ctypes.c_int8), ("y", ctypes.c_int8), ("pad_", ctypes.c_int8),
    ]


SP_DTYPE = np.dtype([
    ("n", "<i8"), ("sum_r", "<i8"), ("sum_g", "<i8"), ("sum_b", "<i8"), ("sum_x", "<i8"), ("sum_y", "<i8"),
    ("mean_r", "<f8"), ("mean_g", "<f8"), ("mean_b", "<f8"), ("mean_x", "<f8"), ("mean_y", "<f8"),
    ("init_size", "<i4"), ("alive", "i1"), ("active", "i1"), ("y", "i1"), ("pad_", "i1"),
])
assert SP_DTYPE.itemsize == ctypes.sizeof(rapid_sp_stat)


class rapid_run_info(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("batch", ctypes.c_uint32), ("H", ctypes.c_uint32), ("W", ctypes.c_uint32),
        ("n_superpixels", ctypes.c_uint32), ("n_stages", ctypes.c_uint32), ("sweeps", ctypes.c_uint32),
        ("grid_rows", ctypes.c_uint32), ("grid_cols", ctypes.c_uint32),
        ("stage_nbx", ctypes.c_uint32 * MAX_STAGES), ("stage_nby", ctypes.c_uint32 * MAX_STAGES),
        ("stage_tiles", ctypes.c_uint64 * MAX_STAGES),
        ("stage_active_tiles", ctypes.c_uint64 * MAX_STAGES),
        ("stage_victims", ctypes.c_uint64 * MAX_STAGES),
        ("stage_merges", ctypes.c_uint64 * MAX_STAGES),
        ("stage_sweeps_run", ctypes.c_uint64 * MAX_STAGES),
        ("stage_window_blocks", ctypes.c_uint64 * MAX_STAGES),
        ("alive", ctypes.c_uint64), ("active", ctypes.c_uint64),
        ("phase", ctypes.c_uint64 * (MAX_STAGES * MAX_SWEEPS * 4 * NCNT)),
    ]

    def counters(self):
        return np.ctypeslib.as_array(self.phase).reshape(MAX_STAGES, MAX_SWEEPS, 4, NCNT).copy()


class rapid_profile(ctypes.Structure):
    _fields_ = [
        ("launches", ctypes.c_uint64 * (NK * MAX_STAGES)),
        ("ms", ctypes.c_double * (NK * MAX_STAGES)),
        ("total_launches", ctypes.c_uint64),
    ]

    def ms_array(self):
        return np.ctypeslib.as_array(self.ms).reshape(NK, MAX_STAGES).copy()

    def launch_array(self):
        return np.ctypeslib.as_array(self.launches).reshape(NK, MAX_STAGES).copy()


class rapid_quality_result(ctypes.Structure):
    _fields_ = [("ue", ctypes.c_double), ("br", ctypes.c_double), ("pixels", ctypes.c_uint64),
                ("leak_px", ctypes.c_uint64), ("gt_boundary_px", ctypes.c_uint64), ("covered_px", ctypes.c_uint64),
                ("pairs", ctypes.c_uint64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` or "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    L.rapid_init.argtypes = [ctypes.POINTER(vp), ctypes.c_int, u64, u64]
    L.rapid_segment.argtypes = [vp, vp, i32, i32, ctypes.POINTER(rapid_params), vp, vp]
    L.rapid_segment_host.argtypes = [vp, vp, i32, i32, ctypes.POINTER(rapid_params), vp, vp]
    L.rapid_segment_host_stream.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), i32, i32, i32,
                                            ctypes.POINTER(rapid_params), vp]
    L.rapid_stats.argtypes = [vp, vp, u64, ctypes.POINTER(rapid_run_info)]
    L.rapid_quality.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, ctypes.POINTER(rapid_quality_result), vp]
    L.rapid_set_profiling.argtypes = [vp, ctypes.c_int]
    L.rapid_get_profile.argtypes = [vp, ctypes.POINTER(rapid_profile)]
    L.rapid_free.argtypes = [vp]
    L.rapid_free.restype = None
    L.rapid_status_string.argtypes = [ctypes.c_int]
    L.rapid_status_string.restype = ctypes.c_char_p
    L.rapid_last_error.argtypes = [vp]
    L.rapid_last_error.restype = ctypes.c_char_p
    L.rapid_debug_stop.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.rapid_debug_map.argtypes = [vp, vp, u64, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    for f in ("rapid_init", "rapid_segment", "rapid_segment_host", "rapid_segment_host_stream", "rapid_quality",
              "rapid_stats",
              "rapid_set_profiling", "rapid_get_profile", "rapid_debug_stop", "rapid_debug_map"):
        getattr(L, f).restype = ctypes.c_int
    return L


lib = _load()

EXPORTS = ("rapid_init", "rapid_segment", "rapid_segment_host", "rapid_segment_host_stream", "rapid_quality",
           "rapid_stats",
           "rapid_set_profiling",
           "rapid_get_profile", "rapid_free", "rapid_status_string", "rapid_last_error",
           "rapid_debug_stop", "rapid_debug_map")


class RapidError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def make_params(p, batch=1) -> rapid_params:
    """Any object with the fields of synth.Params -> rapid_params."""
    o = rapid_params()
    o.struct_size = ctypes.sizeof(rapid_params)
    o.batch = batch
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
            o.proto_rgb[k][ch] = pr[ch]
    o.tau2 = p.tau2
    o.stats_mode = p.stats_mode
    o.y_model = getattr(p, "y_model", 0)
    for i, v in enumerate(getattr(p, "feat_w_q16", [0] * 5)):
        o.feat_w_q16[i] = v
    return o


def load_feature_model(path):
    """SURVEY f2 model file -> rapid_params.feat_w_q16: a JSON object {"bias": b, "w": [w1, w2,
    w3, w4]} of the linear h_theta of Eq. 6 over the features of P:271 (absolute / comparative
    brightness, intra- / extra-region dissimilarity, each in [0, 1] or [-1, 1]), rounded to
    Q16.16.  (Training the model is out of scope: it needs the paper's data.)"""
    import json
    with open(path) as f:
        m = json.load(f)
    w = [m["bias"]] + list(m["w"])
    if len(w) != 5:
        raise ValueError("a feature model has a bias and 4 weights")
    return [int(round(float(v) * 65536)) for v in w]


# ---- same-name wrappers of the C entry points (pointers as ints) ------------------------
def rapid_init(device, max_pixels_total, max_superpixels_total):
    h = ctypes.c_void_p()
    rc = lib.rapid_init(ctypes.byref(h), device, max_pixels_total, max_superpixels_total)
    if rc:
        raise RapidError(rc, "rapid_init")
    return h


def rapid_segment(ctx, image_ptr, H, W, params: rapid_params, labels_ptr, stream_ptr):
    rc = lib.rapid_segment(ctx, image_ptr, H, W, ctypes.byref(params), labels_ptr, stream_ptr)
    if rc:
        raise RapidError(rc, lib.rapid_last_error(ctx).decode())


def rapid_segment_host(ctx, image_ptr, H, W, params: rapid_params, labels_ptr, stream_ptr):
    rc = lib.rapid_segment_host(ctx, image_ptr, H, W, ctypes.byref(params), labels_ptr, stream_ptr)
    if rc:
        raise RapidError(rc, lib.rapid_last_error(ctx).decode())


def rapid_segment_host_stream(ctx, image_ptrs, label_ptrs, H, W, params: rapid_params, stream_ptr):
    n = len(image_ptrs)
    ia = (ctypes.c_void_p * n)(*image_ptrs)
    la = (ctypes.c_void_p * n)(*label_ptrs)
    rc = lib.rapid_segment_host_stream(ctx, ia, la, n, H, W, ctypes.byref(params), stream_ptr)
    if rc:
        raise RapidError(rc, lib.rapid_last_error(ctx).decode())


def rapid_quality(ctx, labels_ptr, gt_ptr, B, H, W, M, eps, stream_ptr) -> rapid_quality_result:
    q = rapid_quality_result()
    rc = lib.rapid_quality(ctx, labels_ptr, gt_ptr, B, H, W, M, eps, ctypes.byref(q), stream_ptr)
    if rc:
        raise RapidError(rc, lib.rapid_last_error(ctx).decode())
    return q


def rapid_stats(ctx, out_ptr, capacity, info: rapid_run_info):
    rc = lib.rapid_stats(ctx, out_ptr, capacity, ctypes.byref(info))
    if rc:
        raise RapidError(rc, lib.rapid_last_error(ctx).decode())


def rapid_free(ctx):
    lib.rapid_free(ctx)


def rapid_status_string(status):
    return lib.rapid_status_string(status).decode()


class Rapid:
    """A context (rapid_ctx) on one CUDA device; torch only provides memory and streams."""

    def __init__(self, device=0, max_pixels=1 << 24, max_superpixels=1 << 16):
        self.device = device
        self.ctx = rapid_init(device, max_pixels, max_superpixels)
        self.last_batch = 1

    def close(self):
        if self.ctx:
            rapid_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def segment(self, image, params, labels=None, stream=None):
        """image: torch.uint8 cuda [B,H,W,3] or [H,W,3] -> torch.int32 [B,H,W] (async on stream)."""
        import torch
        if image.dim() == 3:
            image = image.unsqueeze(0)
        assert image.dtype == torch.uint8 and image.is_cuda and image.is_contiguous()
        B, H, W, C = image.shape
        assert C == 3
        if labels is None:
            labels = torch.empty((B, H, W), dtype=torch.int32, device=image.device)
        assert labels.dtype == torch.int32 and labels.is_contiguous() and labels.shape == (B, H, W)
        st = stream if stream is not None else torch.cuda.current_stream(image.device)
        rapid_segment(self.ctx, image.data_ptr(), H, W, make_params(params, B), labels.data_ptr(),
                      st.cuda_stream)
        self.last_batch = B
        return labels

    def segment_host(self, image, params, labels=None, stream=None):
        """image: numpy u8 [B,H,W,3] (host) -> numpy int32 [B,H,W]; copies are inside the call."""
        img = np.ascontiguousarray(image, dtype=np.uint8)
        if img.ndim == 3:
            img = img[None]
        B, H, W, _ = img.shape
        if labels is None:
            labels = np.empty((B, H, W), dtype=np.int32)
        sp = 0
        if stream is not None:
            sp = stream.cuda_stream
        rapid_segment_host(self.ctx, img.ctypes.data, H, W, make_params(params, B), labels.ctypes.data, sp)
        self.last_batch = B
        return labels

    def segment_host_stream(self, images, params, labels=None, stream=None):
        """images: list of numpy u8 [B,H,W,3] (host; pin them for overlap) -> list of numpy int32
        [B,H,W]; pipelined (the labels of k return while k+1 is copied in and segmented)."""
        imgs = [np.ascontiguousarray(i if i.ndim == 4 else i[None], dtype=np.uint8) for i in images]
        B, H, W, _ = imgs[0].shape
        assert all(i.shape == imgs[0].shape for i in imgs), "all images of a stream share one shape"
        if labels is None:
            labels = [np.empty((B, H, W), dtype=np.int32) for _ in imgs]
        sp = 0 if stream is None else stream.cuda_stream
        rapid_segment_host_stream(self.ctx, [i.ctypes.data for i in imgs], [l.ctypes.data for l in labels], H, W,
                                  make_params(params, B), sp)
        self.last_batch = B
        return labels

    def quality(self, labels, gt, M, eps=2, stream=None):
        """f4: UE / BR of device label maps int32 [B,H,W] (torch, cuda) against device
        ground-truth segment maps of the same shape; returns a dict."""
        import torch
        assert labels.is_cuda and gt.is_cuda and labels.dtype == torch.int32 and gt.dtype == torch.int32
        lab = labels.contiguous() if labels.dim() == 3 else labels.contiguous()[None]
        g = gt.contiguous() if gt.dim() == 3 else gt.contiguous()[None]
        assert lab.shape == g.shape
        B, H, W = lab.shape
        st = stream if stream is not None else torch.cuda.current_stream(lab.device)
        q = rapid_quality(self.ctx, lab.data_ptr(), g.data_ptr(), B, H, W, int(M), int(eps), st.cuda_stream)
        return {"ue": q.ue, "br": q.br, "pixels": q.pixels, "leak": q.leak_px, "gt_boundary": q.gt_boundary_px,
                "covered": q.covered_px, "pairs": q.pairs}

    def stats(self, K=None):
        info = rapid_run_info()
        if K is None:
            K = 0
        out = np.zeros(K, dtype=SP_DTYPE)
        rapid_stats(self.ctx, out.ctypes.data if K else None, K, info)
        return out, info

    def set_profiling(self, level=1):
        lib.rapid_set_profiling(self.ctx, int(level))

    def profile(self):
        pr = rapid_profile()
        rc = lib.rapid_get_profile(self.ctx, ctypes.byref(pr))
        if rc:
            raise RapidError(rc, lib.rapid_last_error(self.ctx).decode())
        return pr

    def debug_stop(self, kind, stage=0, sweep=0, phase=0):
        lib.rapid_debug_stop(self.ctx, kind, stage, sweep, phase)

    def debug_map(self, capacity):
        buf = np.zeros(capacity, dtype=np.int32)
        nbx, nby = ctypes.c_int32(), ctypes.c_int32()
        rc = lib.rapid_debug_map(self.ctx, buf.ctypes.data, capacity, ctypes.byref(nbx), ctypes.byref(nby))
        if rc:
            raise RapidError(rc, lib.rapid_last_error(self.ctx).decode())
        n = self.last_batch * nbx.value * nby.value
        return buf[:n].reshape(self.last_batch, nby.value, nbx.value)

#!/usr/bin/env python
"""Benchmark: Mpixel/s per full RAPID segmentation on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step is one full segmentation (rapid_segment: pyramid, every stage's parity sweeps,
merges, prediction, transitions, final) of the workload's synthetic input, already resident
in HBM.  Default workload: BASELINE.json configs[3] (config 4: 32768x32768, 1 Gpx, M=2^20,
full RAPID pipeline) — the 1-Gpixel configuration the north star's roofline target names.
Inputs are larger than L2 (3.2 GB image, 4.3 GB label map), so no L2 flush is needed.

N>1 (torchrun): every rank segments its own image (different seed): weak scaling, no
collective on the data path ("replicas only").  Timing: W untimed warm-up
steps, then K steps bracketed by barrier + cuda.synchronize, CUDA events on the stream,
max over ranks.  --impl reference times the CPU oracle (the reference arm of this tier) on
a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "Mpixel/s per full segmentation at 1 B200; HBM GB/s fraction of peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--setting", default="rapid", choices=list(synth.SETTINGS),
                    help="SURVEY f1 comparison setting (rapid = the headline workload)")
    ap.add_argument("--sample", type=int, default=8192, help="the bounded CPU sample is side x 2 side px (~15 s of oracle work at 8192)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the untimed f4 UE/BR report")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_for_rank(cfg, rank, setting="rapid"):
    w = synth.with_setting(synth.config(cfg), setting)
    if rank:
        w.seeds = [s + 1000 * rank for s in w.seeds]
    return w


def max_over_ranks(x: float) -> float:
    """Max of a per-rank float over the process group (identity without one).  NCCL groups
    reduce a CUDA tensor, gloo groups (the CPU tests) a host tensor."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kernel_sources_sha16():
    """Hash of the CUDA sources (csrc/*.cu, *.cuh): ties a committed ncu traffic capture to the
    kernels it measured."""
    import hashlib
    d = os.path.join(ROOT, "paper_1704_02083_b200", "csrc")
    h = hashlib.sha256()
    for n in sorted(os.listdir(d)):
        if n.endswith((".cu", ".cuh")):
            with open(os.path.join(d, n), "rb") as f:
                h.update(n.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def config_dict(w, extra=None):
    p = w.params
    d = {"workload": w.name, "batch": w.B, "H": w.H, "W": w.W, "superpixels_per_image": p.n_superpixels,
         "block_sizes": p.block_sizes, "sweeps": p.sweeps,
         "size_mode": ["NONE", "HARD", "MERGE"][p.size_mode],
         "mask_rule": ["OFF", "CLASS", "BSP", "EQ7"][p.mask_rule],
         "stats_mode": ["REUSE", "RECOUNT", "PYRAMID"][p.stats_mode],
        "y_model": ["PROTO", "FEATURES"][getattr(p, "y_model", 0)],
         "l2": "inputs larger than L2 (image %.2f GB, labels %.2f GB); no flush" % (
             w.pixels * 3 / 1e9, w.pixels * 4 / 1e9)}
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(cfg, side, seed_offset=0, setting="rapid"):
    import oracle
    base = synth.config(cfg)
    H, W = min(side, base.H), min(2 * side, base.W)  # side x 2 side: ~15 s of oracle work at 8192
    sw = synth.with_setting(synth.scaled(cfg, H, W, seed_offset=seed_offset), setting)
    img = sw.images()
    t0 = time.perf_counter()
    oracle.segment(img, sw.params)
    dt = time.perf_counter() - t0
    return sw, dt


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


class pinned_to_one_core:
    """Run the (single-threaded) oracle pinned to one host core, as `taskset -c <core>` would
    (BASELINE.md's CPU plan); the previous affinity is restored afterwards."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.old)


def full_oracle_record(cfg):
    """The whole-workload oracle time measured once per round on the GPU box (tools/oracle_full.py
    or the full-size parity test, same single-threaded C oracle, pinned to one core); reported
    next to the live bounded sample, never in place of it."""
    path = os.path.join(ROOT, "profiles", f"oracle_full_cfg{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def cpu_baseline(cfg, side, setting="rapid"):
    model, ncores = cpu_info()
    with pinned_to_one_core() as pin:
        sw, dt = oracle_sample(cfg, side, setting=setting)
    out = {"value": round(sw.pixels / dt / 1e6, 4), "unit": "Mpixel/s", "cores": 1, "kind": "oracle",
           "sample": f"{sw.name}: {sw.H}x{sw.W} px with config {cfg}'s densities and parameters, "
                     f"full pipeline, single-threaded C oracle pinned to core {pin.core}, {dt:.2f} s",
           "cpu_model": model, "host_cores": f"1 of {ncores}"}
    full = full_oracle_record(cfg)
    if full is not None and setting == "rapid":
        out["full_workload"] = full
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    w = synth.with_setting(synth.config(args.config), args.setting)
    times = []
    side = max(1, args.sample // 2)  # side x 2 side per step: ~4 s of oracle work at config 4
    model, ncores = cpu_info()
    with pinned_to_one_core() as pin:
        for i in range(args.warmup + args.steps):
            sw, dt = oracle_sample(args.config, side, seed_offset=0, setting=args.setting)
            if i >= args.warmup:
                times.append(dt)
    px = sw.pixels
    tot = sum(times)
    value = px * len(times) / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mpixel/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot / len(times) * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(w, {"reference_sample": f"{sw.H}x{sw.W} per step"}),
            "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sw.H}x{sw.W} px of config {args.config}'s workload (same "
                                       f"densities/params) per step, single-threaded C oracle pinned to "
                                       f"core {pin.core}",
                             "cpu_model": model, "host_cores": f"1 of {ncores}"},
            "e2e": {"value": round(value, 4), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, index):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def wait_ready(self, timeout=10.0):
        """Block until nvidia-smi has written its first sample (its start-up can take longer than
        a short timed region), so that the samples cover the timed region."""
        if self.p is None:
            return
        t0 = time.time()
        while time.time() - t0 < timeout:
            try:
                if os.path.getsize(self.path) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in open(self.path):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- host link bound
def link_bound(h2d_bytes, d2h_bytes, dev_ms_total, steps, e2e_ms, stream):
    """What bounds the end-to-end number: the host link, measured here with pinned copies of
    1 GiB (best of 3; H2D alone, D2H alone, both at once on two streams), and the pipeline of
    rapid_segment_host_stream over K steps — the first image's copy-in and the last step's
    labels' copy-out cannot overlap anything, every other step costs the slowest of its
    copy-in, its copy-out, both copies through the duplex link, and its segmentation:
        T(K) = t_h2d + t_seg + (K - 1) * max(t_h2d, t_d2h, t_both, t_seg) + t_d2h
    with t_both = (bytes in + bytes out) / duplex bandwidth."""
    import torch
    n = 1 << 30
    hs = torch.empty(n, dtype=torch.uint8).pin_memory()
    hd = torch.empty(n, dtype=torch.uint8).pin_memory()
    da = torch.empty(n, dtype=torch.uint8, device="cuda")
    db = torch.empty(n, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()

    def timed(fn, streams):
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            for st in streams:
                st.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return best

    with torch.cuda.stream(stream):
        t_in = timed(lambda: da.copy_(hs, non_blocking=True), [stream])
        t_out = timed(lambda: hd.copy_(db, non_blocking=True), [stream])

        def both():
            da.copy_(hs, non_blocking=True)
            with torch.cuda.stream(s2):
                hd.copy_(db, non_blocking=True)
        t_both = timed(both, [stream, s2])
    del hs, hd, da, db
    gb = n / 1e9
    h2d, d2h, duplex = gb / t_in, gb / t_out, 2 * gb / t_both  # GB/s
    t_h2d, t_d2h = h2d_bytes / 1e9 / h2d, d2h_bytes / 1e9 / d2h
    t_both = (h2d_bytes + d2h_bytes) / 1e9 / duplex
    t_seg = dev_ms_total / steps / 1e3
    T = t_h2d + t_seg + (steps - 1) * max(t_h2d, t_d2h, t_both, t_seg) + t_d2h
    return {"h2d_gbs": round(h2d, 2), "d2h_gbs": round(d2h, 2), "duplex_gbs": round(duplex, 2),
            "model_ms": round(T * 1e3, 2), "measured_ms": round(e2e_ms, 2),
            "frac": round(T * 1e3 / e2e_ms, 4),
            "how": "pinned 1 GiB torch copies, best of 3 (H2D, D2H, both on two streams); "
                   "T(K) = t_h2d + t_seg + (K-1) max(t_h2d, t_d2h, (in + out) / duplex, t_seg) + t_d2h; "
                   "frac = T(K) / measured"}


# ----------------------------------------------------------------------------- algorithmic bytes
def phase_bytes(info, w, window):
    """SURVEY §8(d) model per K4 launch: 4 B x window blocks + c_s x candidates needing colour
    + 4 B x committed moves.  window[s] = blocks within Chebyshev distance 1 of a block whose
    label can pass the gate (all blocks before prediction)."""
    import paper_1704_02083_b200 as rb
    cnt = info.counters()
    out = {}
    for s, b in enumerate(w.params.block_sizes):
        cs = 3 if b == 1 else 8
        run = int(info.stage_sweeps_run[s])
        byt = 0
        for t in range(run):
            for ph in range(4):
                byt += 4 * window[s] + cs * int(cnt[s, t, ph, rb.C_TOPO]) + 4 * int(cnt[s, t, ph, rb.C_COMMIT])
        out[s] = (byt, run * 4)
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1704_02083_b200 as rb

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    w = workload_for_rank(args.config, rank, args.setting)
    p = w.params
    t0 = time.time()
    host = torch.empty((w.B, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
    w.images(out=host.numpy())
    gen_s = time.time() - t0
    img = host.to(dev)
    labels = torch.empty((w.B, w.H, w.W), dtype=torch.int32, device=dev)
    r = rb.Rapid(local, max_pixels=w.pixels, max_superpixels=w.B * p.n_superpixels)
    stream = torch.cuda.current_stream(dev)

    # untimed: one run with window counting for the algorithmic-bytes model
    r.set_profiling(2)
    r.segment(img, p, labels)
    _, info = r.stats(0)
    window = [int(info.stage_window_blocks[s]) for s in range(len(p.block_sizes))]
    for _ in range(args.warmup):
        r.segment(img, p, labels)
    torch.cuda.synchronize()

    # timed region 1 (the value): K segmentations (one CUDA-graph launch each), CUDA events on
    # the launching stream, no per-kernel events inside
    r.set_profiling(0)
    r.segment(img, p, labels)  # capture + instantiate the graph outside the timed region
    clocks = Clocks(local) if rank == 0 else None
    if clocks:
        clocks.wait_ready()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        r.segment(img, p, labels)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dev_ms = ev0.elapsed_time(ev1)
    ck = clocks.stop() if clocks else None
    # timed region 2 (the per-kernel breakdown and the roofline): the same K segmentations with
    # CUDA events around every launch group, on the launching stream, live
    r.set_profiling(1)
    r.segment(img, p, labels)
    torch.cuda.synchronize()
    prof_ms = np.zeros((rb.NK, rb.MAX_STAGES))
    prof_launch = np.zeros((rb.NK, rb.MAX_STAGES))
    for _ in range(args.steps):
        r.segment(img, p, labels)
        pr = r.profile()  # this segmentation's per-launch-group event times
        prof_ms += pr.ms_array() / args.steps
        prof_launch += pr.launch_array() / args.steps
    total_launches = int(pr.total_launches)
    _, info = r.stats(0)
    # timed region 3 (the phase-set interval): the same K segmentations with events only around
    # each stage's whole phase loop (profiling level 3) — region 2's events between the K3/K4/K5
    # launches break their back-to-back scheduling (~7 us per launch group) and inflate the set
    r.set_profiling(3)
    r.segment(img, p, labels)
    torch.cuda.synchronize()
    set_ms_coarse = np.zeros(rb.MAX_STAGES)
    for _ in range(args.steps):
        r.segment(img, p, labels)
        set_ms_coarse += r.profile().ms_array()[rb.K_PHASESET] / args.steps
    r.set_profiling(1)

    ms_max = max_over_ranks(dev_ms)
    px_total = w.pixels * world * args.steps
    value = px_total / (ms_max / 1e3) / 1e6

    # end to end through the public host API: every step copies its image from pinned host
    # memory to the device and its labels back (rapid_segment_host_stream: K segmentations
    # pipelined over two device buffer pairs — labels of step k return while step k+1's image
    # is copied in and segmented).  Wall clock and CUDA events around the one call.
    e2e = None
    if not args.no_e2e:
        r.set_profiling(0)
        hls = [torch.empty((w.B, w.H, w.W), dtype=torch.int32).pin_memory() for _ in range(2)]
        hn = host.numpy()
        lab_list = [hls[k & 1].numpy() for k in range(args.steps)]
        r.segment_host_stream([hn] * 2, p, [hls[0].numpy(), hls[1].numpy()])  # warm-up (graph capture)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ee0 = torch.cuda.Event(enable_timing=True)
        ee1 = torch.cuda.Event(enable_timing=True)
        e0 = time.perf_counter()
        ee0.record(stream)
        r.segment_host_stream([hn] * args.steps, p, lab_list)
        ee1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - e0) * 1e3
        e_ms = ee0.elapsed_time(ee1)
        te = max_over_ranks(max(e_ms, wall))
        e2e = {"value": round(w.pixels * world * args.steps / (te / 1e3) / 1e6, 3),
               "unit": "Mpixel/s", "h2d_bytes_per_step": w.pixels * 3, "d2h_bytes_per_step": w.pixels * 4,
               "api": "rapid_segment_host_stream (pinned host buffers; H2D, D2H and compute overlapped "
                      "across consecutive steps)"}
        e2e["link"] = link_bound(w.pixels * 3, w.pixels * 4, ms_max, args.steps, te, stream)
        r.set_profiling(1)

    # segmentation quality of this step's labels against the generator's
    # ground-truth segments, on the GPU (rapid_quality), untimed
    quality = None
    if not args.no_quality and rank == 0:
        gt = torch.from_numpy(w.segments()).to(dev)
        r.segment(img, p, labels)
        quality = {f"eps{e}": {k: (round(v, 6) if isinstance(v, float) else v)
                               for k, v in r.quality(labels, gt, p.n_superpixels, e).items()} for e in (0, 2)}
        quality["gt"] = "synth ground truth: tissue Voronoi regions, background cells, nuclei blobs"
        del gt

    if rank == 0:
        peak, peak_src = peaks()
        pb = phase_bytes(info, w, window)
        # Dominant kernel: the K4 sweep (k_sweep: boundary-set driven scan + evaluate) at the
        # pixel stage (the last stage).  Algorithmic bytes per launch: the label
        # reads of the phase's window, 4 B x window blocks, plus the colour reads of the
        # topology-passing candidates, 3 B each.  Label writes (4 B x commits) belong to K5 and
        # enter the phase-set figure below.
        ps = len(p.block_sizes) - 1
        runs = int(info.stage_sweeps_run[ps]) * 4
        cnt = info.counters()
        topo_ps = sum(int(cnt[ps, t, ph, rb.C_TOPO]) for t in range(int(info.stage_sweeps_run[ps])) for ph in range(4))
        sweep_bytes = 4 * window[ps] * runs + 3 * topo_ps
        sweep_ms = float(prof_ms[rb.K_PROPOSE][ps])
        sweep_launch = int(prof_launch[rb.K_PROPOSE][ps])
        steps_ms = float(prof_ms[[rb.K_PYRAMID, rb.K_SNAPSHOT, rb.K_PROPOSE, rb.K_COMMIT, rb.K_MERGE, rb.K_PREDICT,
                                  rb.K_TRANSITION, rb.K_FINAL, rb.K_EVAL]].sum())
        achieved = sweep_bytes / (sweep_ms / 1e3) / 1e9 if sweep_ms > 0 else 0.0
        traffic, traffic_note = None, "no ncu capture committed"
        tfile = os.path.join(ROOT, "profiles", "sweep_traffic.json")
        if os.path.exists(tfile):  # ncu dram bytes of the pixel-stage k_sweep launches (committed capture)
            with open(tfile) as f:
                tj = json.load(f)
            if tj.get("kernel_sources_sha16") == kernel_sources_sha16():
                traffic = tj.get("dram_bytes_per_launch")
                traffic_note = f"ncu capture of these kernel sources ({tj.get('source')})"
            else:
                traffic_note = "stale: the committed ncu capture predates the current kernel sources"
        all_bytes = sum(v[0] for v in pb.values())
        phase_ms_nested = float(prof_ms[rb.K_PHASESET].sum())  # with region 2's inner events
        phase_ms = float(set_ms_coarse.sum())
        # per stage: K4 alone and the per-phase set, bytes per the same model
        per_stage = []
        for st, b in enumerate(p.block_sizes):
            runs_s = int(info.stage_sweeps_run[st]) * 4
            cs = 3 if b == 1 else 8
            topo_s = int(cnt[st, :, :, rb.C_TOPO].sum())
            k4_bytes = 4 * window[st] * runs_s + cs * topo_s
            k4_ms = float(prof_ms[rb.K_PROPOSE][st])
            set_ms = float(set_ms_coarse[st])
            per_stage.append({
                "b": b, "phases": runs_s, "window_blocks": window[st],
                "k4_ms": round(k4_ms, 3), "k4_GB": round(k4_bytes / 1e9, 4),
                "k4_frac": round(k4_bytes / (k4_ms / 1e3) / 1e9 / peak, 4) if k4_ms > 0 else None,
                "k3_ms": round(float(prof_ms[rb.K_SNAPSHOT][st]), 3), "k5_ms": round(float(prof_ms[rb.K_COMMIT][st]), 3),
                "set_ms": round(set_ms, 3), "set_GB": round(pb[st][0] / 1e9, 4),
                "set_frac": round(pb[st][0] / (set_ms / 1e3) / 1e9 / peak, 4) if set_ms > 0 else None})
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_note,
                "phase_set_frac": round(all_bytes / (phase_ms / 1e3) / 1e9 / peak, 4) if phase_ms > 0 else None,
                "kernel": f"k_sweep (K4: boundary-set driven scan + evaluate), pixel stage ({sweep_launch} launches/step)",
                "bytes_per_launch": round(sweep_bytes / max(1, sweep_launch)),
                "avg_launch_ms": round(sweep_ms / max(1, sweep_launch), 4),
                "share_of_step": round(sweep_ms / max(1e-9, steps_ms), 4), "peak_source": peak_src,
                "bytes_model": "4 B x blocks within Chebyshev distance 1 of a block with an active label "
                               "+ 3 B x topology-passing candidates, per phase",
                "phase_set": {"GBps": round(all_bytes / (phase_ms / 1e3) / 1e9, 1) if phase_ms > 0 else None,
                              "frac": round(all_bytes / (phase_ms / 1e3) / 1e9 / peak, 4) if phase_ms > 0 else None,
                              "ms_per_step": round(phase_ms, 3),
                              "ms_per_step_with_inner_events": round(phase_ms_nested, 3),
                              "timing": "CUDA events around each stage's whole phase loop (profiling level 3: "
                                        "no events between the K3/K4/K5 launches); the per-kernel figures "
                                        "(k3_ms, k4_ms, k5_ms, per_kernel_ms_per_step) come from the pass with "
                                        "events around every launch group, whose phase-set interval is "
                                        "ms_per_step_with_inner_events",
                              "kernels": "K3 snapshot + K4 sweep + K5 commit, all stages",
                              "bytes_model": "4 B x window + c_s x topology-passing candidates + 4 B x commits"},
                "per_stage": per_stage}
        line = {"metric": METRIC, "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
                "data": "synthetic", "config": config_dict(w, {"parallelism": f"replicas{world}",
                                                                 "gen_s": round(gen_s, 1)}),
                "roofline": roof, "e2e": e2e, "gpu_launches": total_launches * args.steps,
                "clocks": ck,
                "per_kernel_ms_per_step": {nm: round(float(prof_ms[k].sum()), 3) for k, nm in enumerate(
                    ["pyramid", "snapshot", "sweep", "commit", "merge", "predict", "transition", "final",
                     "phase_set", "eval"])},
                "stage_sweep_ms": [round(float(x), 3) for x in prof_ms[rb.K_PROPOSE][:len(p.block_sizes)]],
                "stage_sweeps_run": [int(x) for x in info.stage_sweeps_run[:len(p.block_sizes)]],
                "stage_candidates": [int(cnt[s, :, :, rb.C_CAND].sum()) for s in range(len(p.block_sizes))],
                "stage_commits": [int(cnt[s, :, :, rb.C_COMMIT].sum()) for s in range(len(p.block_sizes))],
                "setting": args.setting,
                "quality": quality,
                "alive": int(info.alive), "active": int(info.active)}
        if not args.no_cpu and world == 1:  # (the oracle runs on rank 0 at N = 1 only)
            line["cpu_baseline"] = cpu_baseline(args.config, args.sample, args.setting)
        print(json.dumps(line), flush=True)
    r.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

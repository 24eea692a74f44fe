"""Run the CPU oracle on a whole workload once and report its time and peak RSS (the
cpu_baseline for full config 4, BASELINE.md's plan: single-threaded, pinned with taskset).
Optionally saves labels + sums for a later comparison.

    taskset -c 0 python tools/oracle_full.py --config 4 [--save out.npz]
"""
import argparse
import json
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def cpu_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--side", type=int, default=0)
    ap.add_argument("--save", default="")
    a = ap.parse_args()
    w = synth.scaled(a.config, a.side, a.side) if a.side else synth.config(a.config)
    t0 = time.perf_counter()
    img = w.images()
    gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = oracle.segment(img, w.params)
    dt = time.perf_counter() - t0
    out = {"workload": w.name, "pixels": w.pixels, "oracle_s": round(dt, 2),
           "mpx_s": round(w.pixels / dt / 1e6, 3), "gen_s": round(gen, 1),
           "max_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 2),
           "alive": int(r.sp["alive"].sum()), **cpu_info()}
    if a.save:
        np.save(a.save + "_labels.npy", r.labels)
        np.save(a.save + "_sp.npy", r.sp)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

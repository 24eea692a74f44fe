"""Run N segmentations of a config (for ncu captures / launch lists).

    python tools/profile_one.py [--config 4] [--n 1]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1704_02083_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--side", type=int, default=0, help="scaled sample side (0 = full config)")
ap.add_argument("--window", type=int, default=0, help="count algorithmic window blocks (profiling level 2)")
a = ap.parse_args()
w = synth.config(a.config) if not a.side else synth.scaled(a.config, a.side, a.side)
host = torch.empty((w.B, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
w.images(out=host.numpy())
img = host.cuda()
r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=w.B * w.params.n_superpixels)
if a.window:
    r.set_profiling(2)
for i in range(a.n):
    t0 = time.time()
    lab = r.segment(img, w.params)
    torch.cuda.synchronize()
    print(f"segmentation {i}: {1e3 * (time.time() - t0):.2f} ms", flush=True)
_, info = r.stats(0)
print("active tiles per stage:", list(info.stage_active_tiles)[:len(w.params.block_sizes)],
      "tiles:", list(info.stage_tiles)[:len(w.params.block_sizes)])
print("window blocks per stage:", list(info.stage_window_blocks)[:len(w.params.block_sizes)],
      "blocks:", [int(info.stage_nbx[s]) * int(info.stage_nby[s]) * w.B for s in range(len(w.params.block_sizes))])
print("victims:", list(info.stage_victims)[:6], "merges:", list(info.stage_merges)[:6])
cnt = info.counters()
for s in range(len(w.params.block_sizes)):
    print("stage", s, "cand/topo/prop/srej/commit/crej per sweep:",
          [cnt[s, t].sum(axis=0).tolist() for t in range(w.params.sweeps)])
r.close()

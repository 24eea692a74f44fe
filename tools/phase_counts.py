"""Per-phase device counters of one segmentation (rapid_run_info.phase: gated candidates,
simple-point passes, proposals, size rejections, commits, budget drops) and the active
tiles of every stage.

    python tools/phase_counts.py [--config 4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1704_02083_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
a = ap.parse_args()
w = synth.config(a.config)
img = torch.from_numpy(w.images()).cuda()
r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=w.B * w.params.n_superpixels)
r.segment(img, w.params)
_, info = r.stats(0)
ns = len(w.params.block_sizes)
cnt = info.counters()
print("| stage (b) | active tiles / tiles | victims / merges | sweep.phase: cand / topo / prop / commit |")
print("|---|---|---|---|")
for s in range(ns):
    cells = []
    for t in range(int(info.stage_sweeps_run[s])):
        for ph in range(4):
            c = cnt[s, t, ph]
            cells.append(f"{t}.{ph}: {c[0]}/{c[1]}/{c[2]}/{c[4]}")
    print(f"| {s} ({w.params.block_sizes[s]}) | {info.stage_active_tiles[s]} / {info.stage_tiles[s]} | "
          f"{info.stage_victims[s]} / {info.stage_merges[s]} | "
          + "; ".join(cells) + " |")

"""SURVEY f4 with the paper's §4.2 experiment shape (Fig. "merge"): UE and BR of
CTFTPS with and without RAPID's size-regularity optimisation (HARD vs MERGE size modes, no
mask) for a varied number of superpixels, on synthetic images with config 1's shape (the
BSD500 stand-in), scored on the GPU against the generator's ground truth.

    python tools/quality_regularity.py > profiles/<round>_quality_regularity.md
"""
import copy
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_02083_b200 as rb  # noqa: E402
import synth  # noqa: E402

SEEDS = range(1, 21)  # 20 images (the paper uses 200 BSD500 images)
r = rb.Rapid(0, max_pixels=1 << 20, max_superpixels=1 << 14)
print("| M | size mode | UE (mean) | BR eps=2 (mean) |")
print("|---|---|---|---|")
for M in (100, 200, 400, 800, 1600):
    for mode, name in ((synth.SIZE_HARD, "HARD (CTFTPS)"), (synth.SIZE_MERGE, "MERGE (RAPID regularity)")):
        ue, br = [], []
        for seed in SEEDS:
            w = synth.config(1)
            w.seeds = [seed]
            p = copy.deepcopy(w.params)
            p.n_superpixels = M
            p.lambda_pos_q16 = synth.lambda_pos_default(w.H, w.W, M)
            p.size_mode = mode
            img = torch.from_numpy(w.images()).cuda()
            gt = torch.from_numpy(w.segments()).cuda()
            lab = r.segment(img, p)
            q = r.quality(lab, gt, M, 2)
            ue.append(q["ue"])
            br.append(q["br"])
        print(f"| {M} | {name} | {np.mean(ue):.4f} | {np.mean(br):.4f} |")
r.close()

"""Lower bound of a pixel-stage K4 launch's DRAM traffic at sector granularity: the union of
the 32-B sectors of the 3x3 label windows and of the pixel colours of one phase's gated
boundary candidates, computed with torch on the GPU from the label map at a debug stop.
Compared with ncu's dram__bytes_read of the same launch it separates intrinsic sector
granularity (row-major layout) from re-reads (no reuse across warps / tiles).

    python tools/sector_union.py [--stage 5 --sweep 1 --phase 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_1704_02083_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stage", type=int, default=5)
ap.add_argument("--sweep", type=int, default=1)
ap.add_argument("--phase", type=int, default=1, help="the phase whose candidates are counted")
a = ap.parse_args()
w = synth.config(4)
img = torch.from_numpy(w.images()).cuda()
K = w.B * w.params.n_superpixels
r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=K)
# stop after the phase before it (the map the counted phase reads)
ps, pt = (a.phase - 1, a.sweep) if a.phase > 0 else (3, a.sweep - 1)
r.debug_stop(rb.STOP_PHASE, a.stage, pt, ps)
lab = r.segment(img, w.params)
torch.cuda.synchronize()
sp, _ = r.stats(K)
act = torch.from_numpy(sp["active"].astype("bool")).cuda()
L = lab[0].long()
H, W = L.shape
cx, cy = a.phase & 1, a.phase >> 1
bnd = torch.zeros_like(L, dtype=torch.bool)
bnd[1:, :] |= L[1:, :] != L[:-1, :]
bnd[:-1, :] |= L[:-1, :] != L[1:, :]
bnd[:, 1:] |= L[:, 1:] != L[:, :-1]
bnd[:, :-1] |= L[:, :-1] != L[:, 1:]
par = torch.zeros_like(bnd)
par[cy::2, cx::2] = True
C = bnd & par & act[L]
del bnd, par
ncand = int(C.sum())
D = F.max_pool2d(C[None, None].half(), 3, stride=1, padding=1)[0, 0] > 0  # 3x3 windows
win_blocks = int(D.sum())
lab_sectors = int(D.view(H, W // 8, 8).any(-1).sum())
lab64 = int(D.view(H, W // 16, 16).any(-1).sum())
lab128 = int(D.view(H, W // 32, 32).any(-1).sum())
del D
ys, xs = C.nonzero(as_tuple=True)
off = (ys * W + xs) * 3
sec = torch.cat([off >> 5, (off + 2) >> 5]).unique()
img_sectors = int(sec.numel())
img64 = int(torch.cat([off >> 6, (off + 2) >> 6]).unique().numel())
img128 = int(torch.cat([off >> 7, (off + 2) >> 7]).unique().numel())
print(f"stage {a.stage} sweep {a.sweep} phase {a.phase}: candidates {ncand}")
print(f"  window blocks (union) {win_blocks} = {4 * win_blocks / 1e6:.1f} MB at 4 B")
print(f"  label sectors (union) {lab_sectors} = {32 * lab_sectors / 1e6:.1f} MB")
print(f"  image sectors (union) {img_sectors} = {32 * img_sectors / 1e6:.1f} MB (3 B x candidates = {3 * ncand / 1e6:.1f} MB)")
print(f"  lower bound {32 * (lab_sectors + img_sectors) / 1e6:.1f} MB")
print(f"  at 64-B granularity: labels {64 * lab64 / 1e6:.1f} MB + image {64 * img64 / 1e6:.1f} MB = {64 * (lab64 + img64) / 1e6:.1f} MB")
print(f"  at 128-B granularity: labels {128 * lab128 / 1e6:.1f} MB + image {128 * img128 / 1e6:.1f} MB = {128 * (lab128 + img128) / 1e6:.1f} MB")

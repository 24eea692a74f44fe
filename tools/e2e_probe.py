"""Time rapid_segment_host_stream over K = 1, 2, 4, 8 consecutive config-4 segmentations
(pinned host buffers) to see the per-step increment of the pipelined host API.

    python tools/e2e_probe.py [--config 4]
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
a = ap.parse_args()
w = synth.config(a.config)
host = torch.empty((w.B, w.H, w.W, 3), dtype=torch.uint8).pin_memory()
w.images(out=host.numpy())
hls = [torch.empty((w.B, w.H, w.W), dtype=torch.int32).pin_memory() for _ in range(2)]
r = rb.Rapid(0, max_pixels=w.pixels, max_superpixels=w.B * w.params.n_superpixels)
r.set_profiling(0)
hn = host.numpy()
r.segment_host_stream([hn] * 2, w.params, [hls[0].numpy(), hls[1].numpy()])
for K in (1, 2, 4, 8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r.segment_host_stream([hn] * K, w.params, [hls[k & 1].numpy() for k in range(K)])
    torch.cuda.synchronize()
    print(f"K={K}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
t0 = time.perf_counter()
r.segment_host(hn, w.params, hls[0].numpy())
print(f"segment_host: {1e3 * (time.perf_counter() - t0):.1f} ms")

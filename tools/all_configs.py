"""Measure every BASELINE.json config on one GPU: GPU Mpx/s per segmentation (bench.py), the
sweep roofline fraction, and the single-threaded oracle's Mpx/s on the same input (configs
1-3 and 5 in full here; config 4's whole-run oracle time from profiles/oracle_full_cfg4.json).
Prints a markdown table.

    python tools/all_configs.py > profiles/<round>_all_configs.md
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (the oracle is reached only through bench.py's reference arm)


def oracle_full(cfg):
    """The single-threaded oracle on the whole workload of config `cfg`, through bench.py's
    reference arm (one step, no warm-up, the sample as large as the config: pinned to one core)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", str(cfg),
                          "--sample", "65536", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    return d["value"], d["ms_per_step"] / 1e3


rows = []
for cfg in (1, 2, 3, 4, 5):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "10",
                          "--warmup", "3", "--no-e2e", "--no-cpu"], capture_output=True, text=True, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    if cfg == 4:  # the whole config-4 oracle run (106 s, 25 GB) is measured once per round
        with open(os.path.join(ROOT, "profiles", "oracle_full_cfg4.json")) as f:
            full = json.load(f)
        rows.append((cfg, d, full["value"], "full, tools/oracle_full.py", full["seconds"]))
        continue
    mpx, dt = oracle_full(cfg)
    rows.append((cfg, d, mpx, "full", dt))

print("| config | workload | GPU ms / segmentation | GPU Mpx/s | k_sweep frac (pixel stage) | "
      "phase-set frac | oracle Mpx/s (1 core) | oracle input |")
print("|---|---|---|---|---|---|---|---|")
for cfg, d, omp, what, dt in rows:
    c = d["config"]
    print(f"| {cfg} | {c['batch']}×{c['H']}×{c['W']}, M={c['superpixels_per_image']}, {c['size_mode']}/{c['mask_rule']} | "
          f"{d['ms_per_step']:.3f} | {d['value']:.0f} | {d['roofline']['frac']:.3f} | "
          f"{d['roofline']['phase_set']['frac']:.3f} | {omp:.2f} | {what} ({dt:.1f} s) |")

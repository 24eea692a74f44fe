"""time the paper's comparison settings (Table 1) on this path.

    python tools/ablation.py [--config 4] [--steps 5] > profiles/<round>_ablation.md

Runs bench.py once per setting (rapid, ctftps, multiscale; no e2e / CPU legs) and prints a
markdown table: ms per segmentation, Mpx/s, per-stage sweep time, boundary candidates per stage
(the queue size Q the paper's speedup argument rests on) and commits.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
rows = []
for setting in ("rapid", "rapid_pyramid", "rapid_features", "ctftps", "multiscale"):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(a.config), "--steps",
                          str(a.steps), "--warmup", "3", "--no-e2e", "--no-cpu", "--setting", setting],
                         capture_output=True, text=True, check=True).stdout
    rows.append(json.loads(out.strip().splitlines()[-1]))
print(f"# f1 comparison settings, config {a.config} ({rows[0]['config']['H']}x{rows[0]['config']['W']}, "
      f"M = {rows[0]['config']['superpixels_per_image']}), one B200\n")
print("| setting | size / mask / stats | ms per segmentation | Mpx/s | sweep ms per stage | "
      "candidates per stage (M) | commits per stage (k) | UE | BR (eps 0 / 2) |")
print("|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    print(f"| {d['setting']} | {c['size_mode']} / {c['mask_rule']} / {c['stats_mode']} | {d['ms_per_step']:.2f} | "
          f"{d['value']:.0f} | {', '.join(f'{x:.2f}' for x in d['stage_sweep_ms'])} | "
          f"{', '.join(f'{x / 1e6:.1f}' for x in d['stage_candidates'])} | "
          f"{', '.join(f'{x / 1e3:.0f}' for x in d['stage_commits'])} | "
          f"{d['quality']['eps2']['ue']:.4f} | {d['quality']['eps0']['br']:.4f} / {d['quality']['eps2']['br']:.4f} |")
base = {d["setting"]: d["ms_per_step"] for d in rows}
print(f"\nRAPID vs CTFTPS: {base['ctftps'] / base['rapid']:.2f}x; RAPID vs multi-scale CTFTPS: "
      f"{base['multiscale'] / base['rapid']:.2f}x (the paper reports 4x and 13x on a 12-core Xeon, "
      "Table 1 / P:316, P:352: context, not a target).")
